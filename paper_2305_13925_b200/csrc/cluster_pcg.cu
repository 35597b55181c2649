// Fused persistent-state Jac-PCG / CG for the large-K rzf path (complex64,
// K = 128) on a 2-CTA thread-block cluster.
//
// One cluster per realization b solves A X = I (K identity right-hand sides,
// w0 = 0, T iterations; textbook Jac-PCG linsolve.py:259-294, Algorithm 1 and
// CG linsolve.py:217-256) and then forms GX = (A - xi I) X and the ||F||^2
// partials (precoder.py:64-70 with F = H X, metrics.py:35-44 with B = beta GX),
// the same outputs as tc_pcg + tc_gx (gemm_tc.cu) without any HBM round trip
// of the solver state.
//
// Real embedding (2K = 256 components, interleaved re/im): A'' (2K x 2K),
// P, X, R (2K x K: column j = RHS j).  The 3xFP16 split of A'' (hi + lo,
// 256 KiB) does not fit one SM's shared memory, so the pair splits it by
// rows: CTA c holds component rows [128c, 128c + 128) of A'' in its TMEM
// (the tensor-core A operand, hi and lo) and owns the same rows of R (TMEM),
// X (smem) and P (registers).  Each iteration:
//   - the column maxima of P are combined across the pair through DSMEM
//     (per-column power-of-two scale for the fp16 split, as in the fused
//     kernel: converged columns keep their relative precision);
//   - each CTA writes its 128 rows of the scaled, split P into its B operand
//     tile and bulk-copies them (cp.async.bulk shared::cta -> shared::cluster,
//     mbarrier completion) into the peer's, so each holds all 2K rows;
//   - Q_c = A''_c P on the tensor cores (48 tcgen05.mma, M = 128, N = K, from
//     TMEM x smem), one elected thread per CTA;
//   - per-column curvature and rz partials are summed over the CTA's rows in
//     a fixed order, exchanged through DSMEM (st.async completing on the
//     peer's mbarrier) and added rank 0 + rank 1 in both CTAs: the scalars
//     are bit-identical in the pair and deterministic.
// No cluster-wide barrier inside the solve: every exchange completes on an
// mbarrier of the receiver, and the causal chain of the exchanges orders each
// buffer's reuse (see pair_round / product).
//
// Scaling: A'' = sa A with sa = 2^e (diag(A'') < 2^14); iterates are those of
// the unscaled recurrence up to rounding (X = sa X'').
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "xl_common.cuh"

namespace xl {
namespace cpcg {

#include "tc_ptx.cuh"

constexpr int KU = 128;           // users (RHS columns)
constexpr int NC = 2 * KU;        // real components (K-dim of the products)
constexpr int ROWS = 128;         // component rows per CTA
constexpr int NT = 512;           // 16 warps: lane quadrant q = warp & 3, column block h = warp >> 2
constexpr int JH = 32;            // RHS columns per thread
constexpr int SBOA = NC * 16;     // K-major A staging tile: 8-row group stride
constexpr int LBOB = KU * 16;     // MN-major B tile (P / X): 8-K group stride
constexpr int PART = (NC / 8) * LBOB;  // one B tile (hi or lo): 64 KiB
static_assert(PART == (ROWS / 8) * SBOA, "A staging reuses the B tiles");
constexpr int OFF_PB = 0;               // B operand hi, lo (A'' staging before the solve)
constexpr int OFF_XS = 2 * PART;        // X'' (fp32, column-major 128 rows x K)
constexpr int OFF_SMALL = OFF_XS + ROWS * KU * 4;
// TMEM columns
constexpr uint32_t T_AH = 0, T_AL = 128, T_Q = 256, T_R = 384;
constexpr uint32_t ID_P = idesc(128, KU, 0, 1);  // A'' K-major (TMEM), P MN-major (smem)

struct Small {
  uint64_t q_full, cp_done;
  uint64_t pbar;                  // the peer's rows of the B tile have landed (bulk copy)
  uint64_t xbar[2];               // the peer's column partials have landed (per round parity)
  uint32_t tmem_slot;
  int zero_diag, not_hpd, pad;
  float red[4 * 4 * JH];          // per (quadrant, column block) column partials
  float xin[2][KU];               // the peer's column partials [round parity][column]
  alignas(16) float coef[2][KU];  // alpha, beta
  alignas(16) float spx[KU];      // per-column B scale 2^e ...
  alignas(16) float spy[KU];      // ... and 2^-e
  float rzs[KU];
  float cdg[KU];                  // Re diag(A) (includes xi)
  float mred[16];
  double dred[16];
};
constexpr int SMEM = OFF_SMALL + (int)sizeof(Small);
static_assert(SMEM <= 227 * 1024, "cluster PCG smem");

struct Params {
  const float2* A;  // [B][K][K] regularized Gram (Hermitian, xi on the diagonal)
  int64_t B;
  int T, method, variant;
  double xi;
  const double* xi_b;
  float2* X;        // [B][K][K]
  float2* GX;       // [B][K][K] (A - xi I) X
  double* part;     // [B][2] Re tr(X^H GX) per CTA
  int32_t* status;  // [B]
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// 4 bytes into the peer's smem, completing tx bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_f32(uint32_t a, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}
// bulk copy (async proxy) of local smem into the peer's, completing on the peer's mbarrier
__device__ __forceinline__ void bulk_s2s(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// per-thread column values -> red[(q * 4 + h) * JH + j] (warp transpose-reduce)
template <bool MAX = false>
__device__ __forceinline__ void col_partials(float (&v)[JH], float* red, int q, int h) {
  const int lane = threadIdx.x & 31;
  const float t = warp_transpose_reduce<JH, MAX>(v);
  red[(q * 4 + h) * JH + lane] = t;
}
// the CTA's partial of column j (fixed quadrant order)
template <bool MAX = false>
__device__ __forceinline__ float col_total(const float* red, int j) {
  const int h = j / JH, jj = j % JH;
  const float a = red[(0 * 4 + h) * JH + jj], b = red[(1 * 4 + h) * JH + jj];
  const float c = red[(2 * 4 + h) * JH + jj], d = red[(3 * 4 + h) * JH + jj];
  return MAX ? fmaxf(fmaxf(a, b), fmaxf(c, d)) : ((a + b) + c) + d;
}
__device__ __forceinline__ void lds8(const float* a, float (&o)[8]) {
  const float4 x = reinterpret_cast<const float4*>(a)[0], y = reinterpret_cast<const float4*>(a)[1];
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w; o[4] = y.x; o[5] = y.y; o[6] = y.z; o[7] = y.w;
}

// One cross-CTA round n (threads j < K; the caller synchronises the CTA after
// it): the CTA partial of column j goes to the peer's slot xin[n & 1][j] by
// st.async, completing on the peer's xbar[n & 1]; the pair total adds rank 0's
// partial first, so both CTAs hold identical bits.  Slot reuse is safe without
// a cluster barrier: a CTA sends round n + 2 only after receiving the peer's
// round n + 1, which the peer sends after reading round n.
template <bool MAX>
__device__ __forceinline__ float pair_round(Small* sm, uint32_t rank, uint32_t peer_xin, uint32_t peer_xbar, uint32_t n,
                                            int j) {
  if (j >= KU) return 0.0f;
  const int par = n & 1;
  const float own = col_total<MAX>(sm->red, j);
  if (j == 0) mbar_expect_tx(&sm->xbar[par], KU * 4);
  st_async_f32(peer_xin + 4u * (uint32_t)(par * KU + j), own, peer_xbar + 8u * par);
  mbar_wait(&sm->xbar[par], (n >> 1) & 1);
  const float other = sm->xin[par][j];
  const float a = rank == 0 ? own : other, b = rank == 0 ? other : own;
  return MAX ? fmaxf(a, b) : a + b;
}

// Write this thread's JH columns of component row rg (column j scaled by
// spx[j]) as 16-B core-matrix rows of the split MN-major B tile.
__device__ __forceinline__ void write_b(const float (&v)[JH], const float* spx, int rg, int h, uint8_t* bh) {
#pragma unroll
  for (int g = 0; g < JH / 8; ++g) {
    float sv[8];
    lds8(spx + h * JH + 8 * g, sv);
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split2(v[8 * g + 2 * i] * sv[2 * i], v[8 * g + 2 * i + 1] * sv[2 * i + 1], hw[i], lw[i]);
    const int o = (rg >> 3) * LBOB + ((h * JH) / 8 + g) * 128 + (rg & 7) * 16;
    const uint4 H4 = make_uint4(hw[0], hw[1], hw[2], hw[3]), L4 = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    *reinterpret_cast<uint4*>(bh + o) = H4;
    *reinterpret_cast<uint4*>(bh + PART + o) = L4;
  }
}

// Q = A'' B (3xFP16: hi*hi + hi*lo + lo*hi), A'' in TMEM, B in smem; one thread.
// warp-collective: all 32 lanes call it, tcgen05 ops elect one lane (tc_ptx.cuh)
__device__ __forceinline__ void issue_q(uint32_t tmem, uint32_t ub, uint64_t* bar) {
  tc_after();
#pragma unroll
  for (int s = 0; s < NC / 16; ++s) {
    const uint64_t dbh = sdesc(ub + 2 * s * LBOB, LBOB, 128), dbl = sdesc(ub + PART + 2 * s * LBOB, LBOB, 128);
    mma_ts_w(tmem + T_Q, tmem + T_AH + 8 * s, dbh, ID_P, s != 0);
    mma_ts_w(tmem + T_Q, tmem + T_AH + 8 * s, dbl, ID_P, 1);
    mma_ts_w(tmem + T_Q, tmem + T_AL + 8 * s, dbh, ID_P, 1);
  }
  commit_w(bar);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) cluster_pcg_kernel(Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* pb = smem + OFF_PB;
  float* xs = reinterpret_cast<float*>(smem + OFF_XS);  // xs[col * ROWS + r]
  Small* sm = reinterpret_cast<Small*>(smem + OFF_SMALL);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int64_t b = (int64_t)blockIdx.x >> 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  const int r = 32 * q + lane;                 // local component row (TMEM lane)
  const int rg = (int)rank * ROWS + r;         // global component row
  const int kr = rg >> 1;                      // user
  const bool odd = lane & 1;
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  const uint32_t peer_pb = mapa(su32(pb), peer);
  const uint32_t peer_xin = mapa(su32(&sm->xin[0][0]), peer);
  const uint32_t peer_xbar = mapa(su32(&sm->xbar[0]), peer);
  const uint32_t peer_pbar = mapa(su32(&sm->pbar), peer);

  if (tid == 0) {
    mbar_init(&sm->q_full, 1);
    mbar_init(&sm->cp_done, 1);
    mbar_init(&sm->pbar, 1);
    mbar_init(&sm->xbar[0], 1);
    mbar_init(&sm->xbar[1], 1);
    sm->not_hpd = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm->tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const float2* a = p.A + b * (int64_t)KU * KU;
  if (tid < KU) sm->cdg[tid] = a[(int64_t)tid * KU + tid].x;
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;
  const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
  const uint32_t tQ = tl + T_Q + h * JH, tR = tl + T_R + h * JH;

  // ---- scale: diag(A'') = sa diag(A) < 2^14 (|a_ij| <= max diag for HPD A)
  if (warp < KU / 32) {
    const float d = sm->cdg[tid];
    const float m = warp_max(fabsf(d));
    const unsigned z = __ballot_sync(0xffffffffu, use_c && d == 0.0f);  // linsolve.py:205-208
    if (lane == 0) {
      sm->mred[warp] = m;
      sm->mred[8 + warp] = z ? 1.0f : 0.0f;
    }
  }
  __syncthreads();
  if (tid == 0) sm->zero_diag = (sm->mred[8] + sm->mred[9] + sm->mred[10] + sm->mred[11]) > 0.0f;
  const float dmax = fmaxf(fmaxf(sm->mred[0], sm->mred[1]), fmaxf(sm->mred[2], sm->mred[3]));
  const float sa = pow2_scale(dmax, 14);
  const float cr = use_c ? sm->cdg[kr] * sa : 1.0f;
  const float icr = 1.0f / cr;
  const double alpha = p.xi_b ? p.xi_b[b] : p.xi;

  // ---- A'' rows of this CTA -> K-major split staging tile -> TMEM (hi, lo).
  // Row 2i = (Re a_ij, -Im a_ij), row 2i+1 = (Im a_ij, Re a_ij) per column j.
  {
    const float4* arow = reinterpret_cast<const float4*>(a + (int64_t)kr * KU + h * JH);
#pragma unroll 2
    for (int g = 0; g < JH / 4; ++g) {  // 4 complex columns = 8 components = one core-matrix row
      const float4 v0 = __ldg(arow + 2 * g), v1 = __ldg(arow + 2 * g + 1);
      const float re[4] = {v0.x, v0.z, v1.x, v1.z}, im[4] = {v0.y, v0.w, v1.y, v1.w};
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        split2((odd ? im[i] : re[i]) * sa, (odd ? re[i] : -im[i]) * sa, hw[i], lw[i]);
      const int k = 2 * (h * JH + 4 * g);
      const int o = (r >> 3) * SBOA + (k >> 3) * 128 + (r & 7) * 16;
      *reinterpret_cast<uint4*>(pb + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(pb + PART + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  }
  fence_async_smem();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    const uint32_t ua = su32(pb);
#pragma unroll
    for (int s = 0; s < NC / 16; ++s) {
      tmem_cp_w(tmem + T_AH + 8 * s, sdesc(ua + 2 * s * 128, 128, SBOA));
      tmem_cp_w(tmem + T_AL + 8 * s, sdesc(ua + PART + 2 * s * 128, 128, SBOA));
    }
    commit_w(&sm->cp_done);
  }

  // ---- initial state (linsolve.py:224-229, 264-268): x = 0, r = I (Algorithm 1:
  // C^-1 I), m = z, rz per column
  float P[JH], A[JH];
  {
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float rv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int jc = h * JH + c0 + i;
        const float e = (rg == 2 * jc) ? 1.0f : 0.0f;
        rv[i] = (use_c && !textbook) ? e * icr : e;
        P[c0 + i] = textbook ? e * icr : rv[i];
        xs[jc * ROWS + r] = 0.0f;
      }
      tmem_st8(tR + c0, rv);
    }
    if (tid < KU) {
      const float c0 = use_c ? sm->cdg[tid] * sa : 1.0f;
      const float ic = 1.0f / c0;
      sm->rzs[tid] = textbook ? ic : (use_c ? ic * ic : 1.0f);
    }
    tmem_wait_st();
  }
  mbar_wait(&sm->cp_done, 0);  // the staging tile is free for P
  tc_after();
  cluster_sync();  // the peer has started and finished its own staging copy
  uint32_t nr = 0, nq = 0;  // cross-CTA rounds, tensor-core products
  const uint32_t upb = su32(pb);

  // column max of v over the pair -> spx / spy (power-of-two scale, < 2^14)
  auto pair_scale = [&](float (&v)[JH]) {
#pragma unroll
    for (int jj = 0; jj < JH; ++jj) A[jj] = fabsf(v[jj]);
    col_partials<true>(A, sm->red, q, h);
    __syncthreads();
    const float m = pair_round<true>(sm, rank, peer_xin, peer_xbar, nr++, tid);
    if (tid < KU) {
      const float s = pow2_scale(m, 14);
      sm->spx[tid] = s;
      sm->spy[tid] = 1.0f / s;
    }
    __syncthreads();
  };
  // write v (scaled) into the local B tile, bulk-copy this CTA's 128 rows into
  // the peer's tile (they are contiguous: 16 K-groups of LBOB bytes, hi and
  // lo), then Q = A'' v once the peer's rows have landed.  The peer's previous
  // product has finished reading its tile: it sent this iteration's scale
  // partial only after that.
  auto product = [&](const float (&v)[JH]) {
    write_b(v, sm->spx, rg, h, pb);
    fence_async_smem();
    __syncthreads();
    if (warp == 0) {
      constexpr uint32_t HALF = (ROWS / 8) * LBOB;
      const uint32_t off = rank * HALF;
      if (lane == 0) {
        mbar_expect_tx(&sm->pbar, 2 * HALF);
        bulk_s2s(peer_pb + off, upb + off, HALF, peer_pbar);
        bulk_s2s(peer_pb + PART + off, upb + PART + off, HALF, peer_pbar);
      }
      __syncwarp();
      mbar_wait(&sm->pbar, nq & 1);
      issue_q(tmem, upb, &sm->q_full);
    }
    mbar_wait(&sm->q_full, nq & 1);
    ++nq;
    tc_after();
  };

  // Q = A'' P0 for the diagonal P0 (x0 = 0, b = I): column j of A'' times p_jj
  // (every other term of the product is an exact zero), from this thread's row
  // of A in global memory, into the TMEM accumulator in the product's units
  auto first_q = [&]() {
    const float4* arow = reinterpret_cast<const float4*>(a + (int64_t)kr * KU + h * JH);
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float sx[8], q8[8];
      lds8(sm->spx + h * JH + c0, sx);
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const float4 v = __ldg(arow + (c0 + i) / 2);  // columns c0 + i, c0 + i + 1
        const int jc = h * JH + c0 + i;
        const float p0a = use_c ? 1.0f / (sm->cdg[jc] * sa) : 1.0f, p0b = use_c ? 1.0f / (sm->cdg[jc + 1] * sa) : 1.0f;
        q8[i] = ((sa * (odd ? v.y : v.x)) * p0a) * sx[i];
        q8[i + 1] = ((sa * (odd ? v.w : v.z)) * p0b) * sx[i + 1];
      }
      tmem_st8(tQ + c0, q8);
    }
    tmem_wait_st();
  };

  for (int t = 1; t <= p.T; ++t) {
    pair_scale(P);
    if (t == 1) first_q();
    else product(P);
    const float qs = (use_c && !textbook) ? icr : 1.0f;  // Algorithm 1: z = C^-1 P m
    tmem_ld<JH>(tQ, A);
    tmem_wait_ld();
    // curvature m^H z per column (linsolve.py:276)
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float sy[8];
      lds8(sm->spy + h * JH + c0, sy);
#pragma unroll
      for (int i = 0; i < 8; ++i) A[c0 + i] = P[c0 + i] * ((A[c0 + i] * sy[i]) * qs);
    }
    col_partials(A, sm->red, q, h);
    __syncthreads();
    {
      const float curv = pair_round<false>(sm, rank, peer_xin, peer_xbar, nr++, tid);
      if (tid < KU) {  // alpha_j, NotHpd (linsolve.py:277-280)
        const float rzj = sm->rzs[tid];
        const bool act = rzj > 0.0f;
        if (curv <= 0.0f && act) sm->not_hpd = 1;
        sm->coef[0][tid] = act ? rzj / (curv > 0.0f ? curv : 1.0f) : 0.0f;
      }
    }
    __syncthreads();
    // w += alpha m, r -= alpha Pm, rz partials (linsolve.py:281-284)
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float qv[8], rv[8], al8[8], sy[8];
      tmem_ld8(tQ + c0, qv);
      tmem_ld8(tR + c0, rv);
      lds8(sm->coef[0] + h * JH + c0, al8);
      lds8(sm->spy + h * JH + c0, sy);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int jc = h * JH + c0 + i;
        const float al = al8[i];
        xs[jc * ROWS + r] = xs[jc * ROWS + r] + al * P[c0 + i];
        rv[i] = rv[i] - al * ((qv[i] * sy[i]) * qs);
        const float z = textbook ? rv[i] * icr : rv[i];
        A[c0 + i] = rv[i] * z;
      }
      tmem_st8(tR + c0, rv);
    }
    col_partials(A, sm->red, q, h);
    tmem_wait_st();
    __syncthreads();
    {
      const float rn = pair_round<false>(sm, rank, peer_xin, peer_xbar, nr++, tid);
      if (tid < KU) {  // beta_j, rz update (linsolve.py:284-288)
        const float rzj = sm->rzs[tid];
        sm->coef[1][tid] = rzj > 0.0f ? rn / rzj : 0.0f;
        sm->rzs[tid] = rn;
      }
    }
    __syncthreads();
    // m = z + beta m
#pragma unroll
    for (int c0 = 0; c0 < JH; c0 += 8) {
      float rv[8], be8[8];
      tmem_ld8(tR + c0, rv);
      lds8(sm->coef[1] + h * JH + c0, be8);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float z = textbook ? rv[i] * icr : rv[i];
        P[c0 + i] = z + be8[i] * P[c0 + i];
      }
    }
  }

  // ---- GX = A X - xi X without another product: the recursively updated
  // residual is r = I - A X (textbook / CG) or C^-1 (I - A X) (Algorithm 1),
  // so A X = I - C r (C = I unless Algorithm 1); X = sa X''
#pragma unroll
  for (int jj = 0; jj < JH; ++jj) P[jj] = xs[(h * JH + jj) * ROWS + r];
  tmem_ld<JH>(tR, A);
  tmem_wait_ld();
  double fro = 0.0;
  const double xsa = alpha * (double)sa;
  const float crr = (use_c && !textbook) ? cr : 1.0f;
#pragma unroll
  for (int jj = 0; jj < JH; ++jj) {
    const float e = (rg == 2 * (h * JH + jj)) ? 1.0f : 0.0f;
    const float g = (float)((double)(e - crr * A[jj]) - xsa * (double)P[jj]);
    A[jj] = g;
    fro += (double)(P[jj] * sa) * (double)g;  // Re tr(X^H GX), X = sa X''
  }
  // row-major complex outputs: lanes (2m, 2m+1) hold (Re, Im) of user kr;
  // the even lane stores column pairs 4n, 4n+1 and the odd lane 4n+2, 4n+3
  float2* xo = p.X + b * (int64_t)KU * KU + (int64_t)kr * KU + h * JH;
  float2* go = p.GX + b * (int64_t)KU * KU + (int64_t)kr * KU + h * JH;
#pragma unroll
  for (int jp = 0; jp < JH; jp += 2) {
    const float x0 = P[jp] * sa, x1 = P[jp + 1] * sa, g0 = A[jp], g1 = A[jp + 1];
    const float ox0 = __shfl_xor_sync(0xffffffffu, x0, 1), ox1 = __shfl_xor_sync(0xffffffffu, x1, 1);
    const float og0 = __shfl_xor_sync(0xffffffffu, g0, 1), og1 = __shfl_xor_sync(0xffffffffu, g1, 1);
    if (((jp >> 1) & 1) == (odd ? 1 : 0)) {
      const float4 xv = odd ? make_float4(ox0, x0, ox1, x1) : make_float4(x0, ox0, x1, ox1);
      const float4 gv = odd ? make_float4(og0, g0, og1, g1) : make_float4(g0, og0, g1, og1);
      *reinterpret_cast<float4*>(xo + jp) = xv;
      *reinterpret_cast<float4*>(go + jp) = gv;
    }
  }
  fro = warp_sum(fro);
  if (lane == 0) sm->dred[warp] = fro;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += sm->dred[w];
    p.part[2 * b + rank] = s;
    if (rank == 0) {
      if (sm->zero_diag) p.status[b] = XL_STATUS_SPLITTING;
      else if (sm->not_hpd && p.status[b] == 0) p.status[b] = XL_STATUS_NOT_HPD;
    }
  }
  tc_before();
  cluster_sync();  // no DSMEM access may target an exited CTA
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace cpcg

bool cpcg_supported(int K) {
  if (K != cpcg::KU) return false;
  const char* e = getenv("XL_LARGE_K_SOLVER");  // "gemm": the split-GEMM tc_pcg path (A/B, tests)
  return !(e && e[0] == 'g');
}

// X ~= A^{-1}, GX = (A - xi I) X and part[2b], part[2b+1] (sum = Re tr(X^H GX))
// for B realizations of K = 128 (complex64).  status: Splitting / NotHpd as tc_pcg.
int cpcg_solve(int method, int variant, const void* A, int64_t B, int K, int T, double xi, const double* xi_b,
               void* X, void* GX, double* part, int32_t* status, cudaStream_t st) {
  if (K != cpcg::KU) { set_error("cluster PCG: K = %d unsupported", K); return XL_ERR_UNSUPPORTED; }
  if (B > (int64_t)0x3fffffff) { set_error("cluster PCG: batch too large"); return XL_ERR_UNSUPPORTED; }
  cudaFuncSetAttribute(cpcg::cluster_pcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cpcg::SMEM);
  cpcg::Params p{(const float2*)A, B, T, method, variant, xi, xi_b, (float2*)X, (float2*)GX, part, status};
  cpcg::cluster_pcg_kernel<<<(unsigned)(2 * B), cpcg::NT, cpcg::SMEM, st>>>(p);
  return check_launch("cluster_pcg");
}

}  // namespace xl
