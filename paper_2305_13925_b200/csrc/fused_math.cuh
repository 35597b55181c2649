// Math-warp role of the fused tcgen05 precoder (included by fused_tc.cu).
//
// 8 warps = 2 per TMEM lane quadrant; thread (q, h, lane) owns component row
// r = 32q + lane (interleaved re/im of user r/2) and the JH = K/2 right-hand
// side columns of half h.  With 128 registers per thread the PCG state lives
// where it is cheapest:
//   P   (direction)      registers   (needed by every step)
//   X   (iterate)        TMEM cols T_X
//   R   (residual)       TMEM cols T_R
//   Q = A P              TMEM cols T_Q   (tensor-core product)
// Per-column scalars (curvature, rz, alpha, beta) are finalised once per
// column by 64 threads from warp transpose-reduction partials summed over the
// 4 quadrant warps in a fixed order (deterministic), then broadcast via smem.


template <int KU>
__device__ __forceinline__ void math_role(const Params& p, Small* sm, uint8_t* aeh, uint8_t* ael,
                                          uint8_t* pbh, uint8_t* pbl, uint32_t tmem, int nch) {
  using G = Geo<KU>;
  constexpr int NC = G::NC, JH = G::JH, HC = G::HC;
  static_assert(JH % 8 == 0 && HC % 16 == 0, "math tiling");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mw = warp - NCONV;
  const int q = warp & 3, h = mw >> 2;  // TMEM lane quadrant = warp % 4
  const int r = 32 * q + lane;          // component row / output component
  const bool act_row = r < NC;
  const bool quad_act = 32 * q < NC;    // warp-uniform (NC is a multiple of 32)
  const bool odd = lane & 1;
  const int kr = r >> 1;
  const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
  const uint32_t tQ = tl + G::T_Q + h * JH, tX = tl + G::T_X + h * JH, tR = tl + G::T_R + h * JH;
  const bool textbook = (p.method == XL_JACPCG && p.variant == XL_TEXTBOOK);
  const bool use_c = (p.method == XL_JACPCG);
  const int mt = tid - 32 * NCONV;  // 0..255
  const uint32_t uah = su32(aeh), ual = su32(ael), ubh = su32(pbh), ubl = su32(pbl);
  auto stamp = [&](uint32_t kk, int slot) {
    if (XL_TRACE && p.trace && blockIdx.x == 0 && mt == 0 && kk >= (uint32_t)p.trace_k0 && kk < (uint32_t)p.trace_k0 + 8)
      p.trace[(kk - p.trace_k0) * 32 + slot] = clock64();
  };
  uint32_t k = 0, nq = 0, wc = 0;
  uint32_t wuse[2] = {0, 0};
  for (;; ++k) {
    mbar_wait(&sm->bq_full[k & 3], (k >> 2) & 1);  // realization claimed by the producer
    const int64_t b = sm->bq[k & 3];
    if (b < 0) break;
    const double alpha = p.xi_b ? p.xi_b[b] : p.xi;
    mbar_wait(&sm->scale_ready, k & 1);
    const float sz = sm->sz_slot[k & 1];
    mbar_wait(&sm->gram_full, k & 1);
    stamp(k, 0);
    tc_after();
    const float alpha_s = (float)(alpha * (double)sz * (double)sz);

    // ---- (1) Re diag of A' = G[2k][2k] + G[2k+1][2k+1] (same order as below)
    if (quad_act && h == (32 * q) / HC) {
      float v[32];
      tmem_ld16(tl + G::T_GRAM + 32 * q, v);
      tmem_ld16(tl + G::T_GRAM + 32 * q + 16, v + 16);
      tmem_wait_ld();
      float dg = 0.0f;
#pragma unroll
      for (int i = 0; i < 32; ++i) dg = (i == lane) ? v[i] : dg;
      const float pd = __shfl_xor_sync(0xffffffffu, dg, 1);
      if (!odd) sm->cdg[kr] = dg + pd;
    }
    named_sync(BAR_MATH, NMT);
    float dmax = 0.0f;
    bool range_bad = false;  // per entry: fmaxf would drop a NaN (inf - inf in the split)
    for (int kk = 0; kk < KU; ++kk) {
      const float d = sm->cdg[kk] + alpha_s;
      range_bad |= !isfinite(d);
      dmax = fmaxf(dmax, d);
    }
    const float sa = pow2_scale(dmax, 14);  // diag(A'') < 2^14
    const float gd = act_row ? sm->cdg[kr] : 0.0f;
    const float cr = (act_row && use_c) ? (gd + alpha_s) * sa : 1.0f;
    const float icr = 1.0f / cr;

    // ---- (2) A'' split: row 2k = (ar, -ai), row 2k+1 = (ai, ar) per column pair
    // (the smem operand region held Xe(k-1) until the W pass copied it to TMEM)
    if (k >= 1 && !(dbg_bits(p) & 3)) mbar_wait(&sm->xe_consumed, (k - 1) & 1);
#if XL_GRAM2
    // The Gram pass accumulated U = Zh^T (Zh + 2 Zl) (two products instead of
    // three); G = (U + U^T) / 2.  U goes through smem (rows padded to NC + 4
    // floats: conflict-free 16-B row accesses and 4-B column accesses; the
    // buffer spans the A'' and P tiles, both idle here), each thread forms
    // its half-row of G, and the A'' rows are written after everyone's reads.
    {
      constexpr int UP = NC + 4;
      float* ub = reinterpret_cast<float*>(aeh);
      static_assert(NC * UP * 4 <= 2 * G::AEPART + 2 * G::PBPART, "U staging");
      if (quad_act) {
#pragma unroll 1
        for (int c0 = 0; c0 < HC; c0 += 16) {
          float v[16];
          tmem_ld16(tl + G::T_GRAM + h * HC + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            *reinterpret_cast<float4*>(ub + r * UP + h * HC + c0 + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
      }
      named_sync(BAR_MATH, NMT);
      uint32_t hw[HC / 2], lw[HC / 2];
      if (quad_act) {
#pragma unroll
        for (int c0 = 0; c0 < HC; c0 += 4) {
          const float4 own = *reinterpret_cast<const float4*>(ub + r * UP + h * HC + c0);
          const float gv[4] = {own.x, own.y, own.z, own.w};
          float g[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) g[e] = 0.5f * (gv[e] + ub[(h * HC + c0 + e) * UP + r]);
#pragma unroll
          for (int jp = 0; jp < 2; ++jp) {
            const float g0 = g[2 * jp], g1 = g[2 * jp + 1];
            const float p0 = __shfl_xor_sync(0xffffffffu, g0, 1), p1 = __shfl_xor_sync(0xffffffffu, g1, 1);
            float ar = odd ? (p0 + g1) : (g0 + p1);
            const float ai = odd ? (p1 - g0) : (g1 - p0);
            const int jc = (h * HC + c0) / 2 + jp;
            if (jc == kr) ar += alpha_s;
            if (p.dbgA && !odd) {
              const float inv = 1.0f / (sz * sz);
              p.dbgA[(b * KU + kr) * KU + jc] = make_float2(ar * inv, ai * inv);
            }
            split2((odd ? ai : ar) * sa, (odd ? ar : -ai) * sa, hw[c0 / 2 + jp], lw[c0 / 2 + jp]);
          }
        }
      }
      named_sync(BAR_MATH, NMT);  // U reads done before A'' overwrites the buffer
      if (quad_act) {
#pragma unroll
        for (int q8 = 0; q8 < HC / 8; ++q8) {
          const int o = boff<KU>(r, h * HC + 8 * q8);
          *reinterpret_cast<uint4*>(aeh + o) = make_uint4(hw[4 * q8], hw[4 * q8 + 1], hw[4 * q8 + 2], hw[4 * q8 + 3]);
          *reinterpret_cast<uint4*>(ael + o) = make_uint4(lw[4 * q8], lw[4 * q8 + 1], lw[4 * q8 + 2], lw[4 * q8 + 3]);
        }
      }
    }
#else
    if (quad_act) {
#pragma unroll 1
      for (int c0 = 0; c0 < HC; c0 += 16) {
        float v[16];
        tmem_ld16(tl + G::T_GRAM + h * HC + c0, v);
        tmem_wait_ld();
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int jp = 0; jp < 8; ++jp) {
          const float g0 = v[2 * jp], g1 = v[2 * jp + 1];
          const float p0 = __shfl_xor_sync(0xffffffffu, g0, 1), p1 = __shfl_xor_sync(0xffffffffu, g1, 1);
          float ar = odd ? (p0 + g1) : (g0 + p1);
          const float ai = odd ? (p1 - g0) : (g1 - p0);
          const int jc = (h * HC + c0) / 2 + jp;
          if (jc == kr) ar += alpha_s;
          if (p.dbgA && !odd) {
            const float inv = 1.0f / (sz * sz);
            p.dbgA[(b * KU + kr) * KU + jc] = make_float2(ar * inv, ai * inv);
          }
          split2((odd ? ai : ar) * sa, (odd ? ar : -ai) * sa, hw[jp], lw[jp]);
        }
        // two whole 16-B core-matrix rows per thread (8-lane phases contiguous)
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4) {
          const int o = boff<KU>(r, h * HC + c0 + 8 * q4);
          *reinterpret_cast<uint4*>(aeh + o) = make_uint4(hw[4 * q4], hw[4 * q4 + 1], hw[4 * q4 + 2], hw[4 * q4 + 3]);
          *reinterpret_cast<uint4*>(ael + o) = make_uint4(lw[4 * q4], lw[4 * q4 + 1], lw[4 * q4 + 2], lw[4 * q4 + 3]);
        }
      }
    }
#endif
    tc_before();
    fence_async_smem();
    named_sync(BAR_MATH, NMT);  // every thread's Gram TMEM reads are complete
    if (mt == 0) mbar_arrive(&sm->gram_free);  // the next Gram may accumulate
    if (dbg_bits(p) & 1) {
      if (mt == 0) p.status[b] = range_bad ? XL_STATUS_RANGE : 0;
      continue;
    }
    stamp(k, 1);

    // ---- (3) PCG (linsolve.py:217-294), K identity RHS, w0 = 0
    float P[JH], A[JH];
    {
      float xz[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int c0 = 0; c0 < JH; c0 += 8) {
        float rv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jc = h * JH + c0 + i;
          const float e = (act_row && r == 2 * jc) ? 1.0f : 0.0f;
          rv[i] = (use_c && !textbook) ? e * icr : e;
          P[c0 + i] = textbook ? e * icr : rv[i];
        }
        if (quad_act) {
          tmem_st8(tX + c0, xz);
          tmem_st8(tR + c0, rv);
        }
      }
      if (mt < KU) {  // rz_j = r_j^H z_j of the unit residual (linsolve.py:268)
        const float c0 = use_c ? (sm->cdg[mt] + alpha_s) * sa : 1.0f;
        const float ic = 1.0f / c0;
        sm->rzs[mt] = textbook ? ic : (use_c ? ic * ic : 1.0f);
      }
      tmem_wait_st();
    }
    int not_hpd = 0;
    for (int t = 1; t <= p.T; ++t) {
      // (a) per-column power-of-two scale of P for the fp16 split: columns
      // converge at different rates, and a converged column must keep its
      // relative precision (a shared scale flushes it to zero -> curvature 0)
#pragma unroll
      for (int jj = 0; jj < JH; ++jj) A[jj] = fabsf(P[jj]);
      column_partials<JH, true>(A, sm->red, q, h);
      named_sync(BAR_MATH, NMT);
      if (mt < KU) {
        const float s = pow2_scale(column_max<JH>(sm->red, mt), 14);
        sm->spx[mt] = s;
        sm->spy[mt] = 1.0f / s;
      }
      named_sync(BAR_MATH, NMT);
      if (t == 1) stamp(k, 5);
      // (b) Q = A'' P on the tensor core
      if (act_row) write_cols<KU>(P, sm->spx, 1.0f, r, h, pbh, pbl);
      fence_async_smem();
      named_sync(BAR_MATH, NMT);
      if (t == 1) stamp(k, 6);
      if (mt < 32) issue_kxk<KU>(tmem + G::T_Q, uah, ual, ubh, ubl, &sm->q_full);
      mbar_wait(&sm->q_full, nq & 1);
      ++nq;
      if (t == 1) stamp(k, 7);
      tc_after();
      const float qs = (use_c && !textbook) ? icr : 1.0f;  // Algorithm 1: z = C^-1 P m
      if (quad_act) {
        tmem_ld<JH>(tQ, A);
        tmem_wait_ld();
      }
      // (c) curvature m^H z per column
#pragma unroll
      for (int c0 = 0; c0 < JH; c0 += 8) {
        float sy[8];
        lds8(sm->spy + h * JH + c0, sy);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jj = c0 + i;
          A[jj] = A[jj] * sy[i];  // undo the column scale (exact)
          A[jj] = act_row ? P[jj] * (A[jj] * qs) : 0.0f;
        }
      }
      column_partials<JH>(A, sm->red, q, h);
      named_sync(BAR_MATH, NMT);
      if (mt < KU) {  // (d) alpha_j, NotHpd (linsolve.py:276-280)
        const float curv = column_total<JH>(sm->red, mt);
        const float rzj = sm->rzs[mt];
        const bool act = rzj > 0.0f;
        if (curv <= 0.0f && act) not_hpd = 1;
        sm->coef[0][mt] = act ? rzj / (curv > 0.0f ? curv : 1.0f) : 0.0f;
      }
      named_sync(BAR_MATH, NMT);
      if (t == 1) stamp(k, 12);
      // (e) w += alpha m, r -= alpha Pm, rz partials (linsolve.py:281-284)
#pragma unroll
      for (int c0 = 0; c0 < JH; c0 += 8) {
        float qv[8], xv[8], rv[8], al8[8], sy[8];
        if (quad_act) {
          tmem_ld8(tQ + c0, qv);
          tmem_ld8(tX + c0, xv);
          tmem_ld8(tR + c0, rv);
        }
        lds8(sm->coef[0] + h * JH + c0, al8);
        lds8(sm->spy + h * JH + c0, sy);
        if (quad_act) tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float al = al8[i];
          xv[i] = xv[i] + al * P[c0 + i];
          rv[i] = rv[i] - al * ((qv[i] * sy[i]) * qs);
          const float z = textbook ? rv[i] * icr : rv[i];
          A[c0 + i] = act_row ? rv[i] * z : 0.0f;
        }
        if (quad_act) {
          tmem_st8(tX + c0, xv);
          tmem_st8(tR + c0, rv);
        }
      }
      column_partials<JH>(A, sm->red, q, h);  // (d) finished reading red before the last barrier
      tmem_wait_st();
      if (t == 1) stamp(k, 13);
      named_sync(BAR_MATH, NMT);
      if (mt < KU) {  // (f) beta_j, rz update (linsolve.py:284-288)
        const float rn = column_total<JH>(sm->red, mt);
        const float rzj = sm->rzs[mt];
        sm->coef[1][mt] = rzj > 0.0f ? rn / rzj : 0.0f;
        sm->rzs[mt] = rn;
      }
      named_sync(BAR_MATH, NMT);
      if (t == 1) stamp(k, 14);
      // (g) m = z + beta m
#pragma unroll
      for (int c0 = 0; c0 < JH; c0 += 8) {
        float rv[8], be8[8];
        if (quad_act) tmem_ld8(tR + c0, rv);
        lds8(sm->coef[1] + h * JH + c0, be8);
        if (quad_act) tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float be = be8[i];
          const float z = textbook ? rv[i] * icr : rv[i];
          P[c0 + i] = act_row ? z + be * P[c0 + i] : 0.0f;
        }
      }
      if (t == 1) stamp(k, 15);
    }
    tc_before();
    stamp(k, 2);

    // ---- (4) beta, coupling B = beta G X, SINR (precoder.py:64-70, metrics.py:47-58)
    float xm = 0.0f;
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float xv[8];
      if (quad_act) {
        tmem_ld8(tX + c0, xv);
        tmem_wait_ld();
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) xm = act_row ? fmaxf(xm, fabsf(xv[i])) : xm;
    }
    const float sx = pow2_scale(math_max(xm, sm), 14);
    stamp(k, 19);
    if (act_row && h == r / HC) {  // G'' = A'' - sa xi' I: only the diagonal changes
      __half hh, ll;
      split(gd * sa, hh, ll);
      const int o = boff<KU>(r, r);
      *reinterpret_cast<__half*>(aeh + o) = hh;
      *reinterpret_cast<__half*>(ael + o) = ll;
    }
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float xv[8];
      if (quad_act) {
        tmem_ld8(tX + c0, xv);
        tmem_wait_ld();
      }
      if (act_row) {  // X columns c0..c0+7 as one 16-B row segment of the MN-major B tile
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split2(xv[2 * i] * sx, xv[2 * i + 1] * sx, hw[i], lw[i]);
        const int o = (r >> 3) * G::LBOB + ((h * JH + c0) / 8) * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(pbh + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(pbl + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
    fence_async_smem();
    named_sync(BAR_MATH, NMT);
    stamp(k, 20);
    if (mt < 32) issue_kxk<KU>(tmem + G::T_Q, uah, ual, ubh, ubl, &sm->q_full);
    mbar_wait(&sm->q_full, nq & 1);
    ++nq;
    stamp(k, 21);
    tc_after();
    float GX[JH];
    if (quad_act) {
      tmem_ld<JH>(tQ, GX);
      tmem_wait_ld();
    }
    const float isx = 1.0f / sx;
    // kappa = sa sz^2: X_true = kappa X'', G X_true = GX
    const double kappa = (double)sa * (double)sz * (double)sz;
    float part = 0.0f;  // 32-term per-thread partial in fp32, cross-thread sum in fp64
    float rs = 0.0f;
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float xv[8];
      if (quad_act) {
        tmem_ld8(tX + c0, xv);
        tmem_wait_ld();
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float g = act_row ? GX[c0 + i] * isx : 0.0f;
        GX[c0 + i] = g;
        part = act_row ? fmaf(xv[i], g, part) : part;
        // interference summed directly (j != k): total - signal cancels in fp32
        rs += (h * JH + c0 + i == kr) ? 0.0f : g * g;
      }
    }
    const double fro2 = kappa * math_sum_d((double)part, sm);
    stamp(k, 22);
    double beta = 0.0;
    int degenerate = 0;
    if (fro2 > 0.0 && isfinite(fro2)) beta = sqrt(p.power / fro2);
    else degenerate = 1;
    if (act_row) {
      sm->rsq()[h * NC + r] = rs;
#pragma unroll
      for (int jj = 0; jj < JH; ++jj)
        if (h * JH + jj == kr) sm->dgq()[r] = GX[jj];
    }
    const bool any_not_hpd = math_max(not_hpd ? 1.0f : 0.0f, sm) > 0.0f;  // also orders rsq/dgq
    if (mt < 64) {  // warps 4-5: per-user SINR / SE, then a fixed-order warp sum
      double se = 0.0;
      if (mt < KU) {
        const double b2 = beta * beta;
        const float* rsq = sm->rsq();
        const float* dgq = sm->dgq();
        const double intf = b2 * ((double)rsq[2 * mt] + (double)rsq[NC + 2 * mt] +
                                  (double)rsq[2 * mt + 1] + (double)rsq[NC + 2 * mt + 1]);
        const double sig = b2 * ((double)dgq[2 * mt] * dgq[2 * mt] +
                                  (double)dgq[2 * mt + 1] * dgq[2 * mt + 1]);
        const double g = sig / (intf + p.sigma2);  // metrics.py:52-56
        if (p.gamma) p.gamma[b * KU + mt] = g;
        se = log2(1.0 + g);
      }
      se = warp_sum(se);
      if (lane == 0) sm->sse[mt >> 5] = se;
      if (mt == 0) {  // W^T scales for the converters' epilogue, published before xe_ready
        sm->wsc[k & 1][0] = (float)(beta * kappa / ((double)sz * (double)sx));
        sm->wsc[k & 1][1] = (float)(kappa / ((double)sz * (double)sx));
      }
    }
    stamp(k, 23);

    // ---- (5) X out (optional) and Xe = real embedding of X as the A operand of
    //      W^T = Xe^T Z^T: row c2 = 2j: (xr, -xi), row 2j+1: (xi, xr) at cols (2k, 2k+1)
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float xv[8];
      if (quad_act) {
        tmem_ld8(tX + c0, xv);
        tmem_wait_ld();
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float v = xv[i] * sx;
        const float pv = __shfl_xor_sync(0xffffffffu, v, 1);  // partner: xi for even, xr for odd
        const int jc = h * JH + c0 + i;
        if (act_row) {
          if (p.X) reinterpret_cast<float*>(p.X)[((b * KU + kr) * KU + jc) * 2 + (r & 1)] = (float)(kappa * xv[i]);
          // even: v = xr, pv = xi -> row 2jc = (xr, -xi); odd: row 2jc + 1 = (xi, xr)
          uint32_t hw, lw;
          split2(v, odd ? pv : -pv, hw, lw);
          const int o = boff<KU>(2 * jc + (odd ? 1 : 0), 2 * kr);
          *reinterpret_cast<uint32_t*>(aeh + o) = hw;
          *reinterpret_cast<uint32_t*>(ael + o) = lw;
        }
      }
    }
    stamp(k, 28);
    tc_before();
    fence_async_smem();
    named_sync(BAR_MATH, NMT);
    stamp(k, 29);
    if (mt == 0) {
      mbar_arrive(&sm->xe_ready);
      p.sum_se[b] = sm->sse[0] + sm->sse[1];
      p.beta[b] = beta;
      int st = XL_STATUS_OK;
      if (range_bad) st = XL_STATUS_RANGE;
      else if (any_not_hpd) st = XL_STATUS_NOT_HPD;
      else if (degenerate) st = XL_STATUS_DEGENERATE;
      p.status[b] = st;
    }
    stamp(k, 3);
    // The W pass of this realization (TMA re-read, conversion, W^T MMAs and
    // the TMEM -> HBM epilogue) now proceeds on the converter / MMA warps
    // while these warps move on to the next realization.
  }
  (void)nch;
  (void)wc;
  (void)wuse;
}

// W^T epilogue of one chunk (16-warp layout), run by converter warps 0-3
// (TMEM lane quadrant = warp): thread = output component c2 = 32 q + lane, CH
// antennas; 128-B coalesced streaming stores per antenna.  (Staging the tile in
// smem for 1-D bulk stores measured no faster: the per-SM store path, ~32 B per
// cycle, sets the pace, not the issuing warps.)
template <int KU>
__device__ __forceinline__ void w_epilogue(const Params& p, Small* sm, uint32_t tmem, int64_t b, int c,
                                           uint32_t j, uint32_t parity, uint32_t kpar, long long* tr = nullptr) {
  using G = Geo<KU>;
  constexpr int NC = G::NC, CH = G::CH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warps 0-3 = lane quadrants
  const int r = 32 * warp + lane;
  const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16) + (j ? G::T_W1 : G::T_W0);
  mbar_wait(&sm->wfull[j], parity);
  if (XL_TRACE && tr && threadIdx.x == 0) tr[6] = clock64();
  // the math warps published the scales before xe_ready, which these MMAs awaited
  const float wscale = sm->wsc[kpar][0], fscale = sm->wsc[kpar][1];
  tc_after();
  // two halves of CH/2 antennas keep the register footprint at CH/2 (the
  // converter state lives alongside); the buffer is released after the
  // second TMEM load, before its stores
  constexpr int HALF = CH / 2;
  const int64_t o0 = (b * (int64_t)p.M + (int64_t)c * CH) * NC + r;
  float* wp = reinterpret_cast<float*>(p.W) + o0;
  float* fp = p.F ? reinterpret_cast<float*>(p.F) + o0 : nullptr;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    float d[HALF];
    if (32 * warp < NC) {
      tmem_ld<HALF>(tl + hf * HALF, d);
      tmem_wait_ld();
    }
    if (hf == 1) {
      tc_before();
      mbar_arrive(&sm->wfree[j]);
      if (XL_TRACE && tr && threadIdx.x == 0) tr[7] = clock64();
    }
    if (r < NC && !(dbg_bits(p) & 8)) {  // dbg & 8: timing without the W stores
#pragma unroll
      for (int a = 0; a < HALF; ++a) __stcs(wp + (hf * HALF + a) * NC, d[a] * wscale);
      if (fp) {
#pragma unroll
        for (int a = 0; a < HALF; ++a) __stcs(fp + (hf * HALF + a) * NC, d[a] * fscale);
      }
    }
  }
}

// 20-warp layout (K = 64): half of one chunk's W^T epilogue, CH/2 antennas
// starting at a0, TMEM lane quadrant warp & 3; two warps share a quadrant.
template <int KU>
__device__ __forceinline__ void w_epilogue_half(const Params& p, Small* sm, uint32_t tmem, int64_t b, int c,
                                                uint32_t j, uint32_t parity, uint32_t kpar, int a0,
                                                long long* tr = nullptr) {
  using G = Geo<KU>;
  constexpr int NC = G::NC, CH = G::CH, HALF = CH / 2;
  const int q = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int r = 32 * q + lane;
  const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (j ? G::T_W1 : G::T_W0) + a0;
  mbar_wait(&sm->wfull[j], parity);
  if (XL_TRACE && tr && threadIdx.x == 0) tr[6] = clock64();
  const float wscale = sm->wsc[kpar][0], fscale = sm->wsc[kpar][1];
  tc_after();
  float d[HALF];
  if (32 * q < NC) {
    tmem_ld<HALF>(tl, d);
    tmem_wait_ld();
  }
  tc_before();
  mbar_arrive(&sm->wfree[j]);
  if (XL_TRACE && tr && threadIdx.x == 0) tr[7] = clock64();
  if (r < NC && !(dbg_bits(p) & 8)) {
    const int64_t o0 = (b * (int64_t)p.M + (int64_t)c * CH + a0) * NC + r;
    float* wp = reinterpret_cast<float*>(p.W) + o0;
#pragma unroll
    for (int a = 0; a < HALF; ++a) __stcs(wp + a * NC, d[a] * wscale);
    if (p.F) {
      float* fp = reinterpret_cast<float*>(p.F) + o0;
#pragma unroll
      for (int a = 0; a < HALF; ++a) __stcs(fp + a * NC, d[a] * fscale);
    }
  }
}
