// Fused complex64 precoder for small K (K in {16, 32}) with the realization's
// H resident in shared memory: one CTA per realization, two CTAs per SM.
//
//   A = H^H H + xi I        gram_regularized (precoder.py:53-61)
//   Jac-PCG / CG, T iters   linsolve.py:217-294 on the K identity RHS, w0 = 0
//   GX, ||F||^2, beta       precoder.py:64-70 (K x K form)
//   W = beta H X, F = H X   precoder.py:90
//   B = beta GX, SINR, SE   coupling + sinr_eq9 (metrics.py:35-58)
//
// Why not tcgen05 here.  At K <= 32 the persistent tcgen05 kernel
// (fused_tc.cu) is bound by its math role's latency chain (one realization
// per SM at a time, a TMEM round trip and seven barrier rounds per PCG
// iteration).  This kernel splits the work by the unit
// that suits it:
//
//   * Gram and W (the M x 2K x 2K products, ~90% of the flops) on the warp-
//     level tensor cores (mma.sync m16n8k16, fp16 inputs, fp32 accumulate),
//     3xFP16 split like fused_tc.cu: x = hi + lo, hi = fp16(x),
//     lo = fp16(x - hi); W = Zh Xh + Zh Xl + Zl Xh, and the Gram as
//     U = Zh^T Zh + 2 Zh^T Zl, G = (U + U^T) / 2 (symmetric by construction).
//     Operands come from swizzled smem tiles through ldmatrix, with no TMEM
//     round trip, so two CTAs per SM overlap one realization's tensor work
//     with the other's SIMT solve.
//   * The K x K solve in fp32 SIMT, the state of each thread's RG x 1 block
//     of X, R, P, Q in registers (thread = column j, rows ig*RG ..), the
//     column reductions through one shared-memory partial row per warp
//     group (three barriers per iteration).  G is kept without xi (A p =
//     G p + xi p), so GX = G X is an explicit product with no cancellation
//     against xi X at low SNR; P0 is diagonal (x0 = 0, b = I), so the first
//     product is a column scaling: T iterations cost T K x K products.
//
// Scaling: every user column k of Z (its re and im components) is scaled by
// s_k = 2^e_k so that its largest |component| lies in [2^14, 2^15) -- the
// fp16 split then keeps ~22 bits for every column regardless of the gain
// spread between users.  The Gram is unscaled exactly (A_ij = G'_ij / s_i s_j),
// and W uses Xe' = S^-1 X T with a per-output-column power of two t_j.
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "xl_common.cuh"

namespace xl {
namespace fs {

constexpr int NT = 256, NW = NT / 32;

struct Params {
  const float2* H;
  int64_t B;
  int M, method, variant, T;
  double xi;
  const double* xi_b;
  double power, sigma2;
  float2 *W, *F, *X;
  double *beta, *gamma, *sum_se;
  int32_t* status;
};

template <int K>
struct G {
  static constexpr int NC = 2 * K;        // real components (re/im interleaved, as in H)
  static constexpr int RC = NC * 2 / 16;  // 16-B chunks per fp16 row (8 for K = 32, 4 for K = 16)
  static constexpr int RG = K * K / NT;   // solver rows per thread (4 / 1)
  static constexpr int NG = NT / K;       // solver row groups (8 / 16)
  static constexpr int US = NC + 2;       // fp32 U row stride (2-way conflicts on the fragment stores)
  static constexpr int XT_BYTES = (NC * US * 4 > 2 * NC * NC * 2) ? NC * US * 4 : 2 * NC * NC * 2;
  static constexpr int MT = NC / 16, NTL = NC / 8;           // m16 / n8 tiles of a 2K x 2K product
  static constexpr int GNP = K == 32 ? 4 : 2;                // Gram n-tiles per warp
  static constexpr int GWARPS = MT * NTL / GNP;              // Gram warps (8 / 4)
  static_assert(RG * NG == K, "solver mapping");
  static_assert(GWARPS <= NW, "Gram mapping");
};

// (row, 16-B chunk) of a swizzled fp16 tile with RC chunks per row: the 8 rows
// an ldmatrix phase reads at one chunk land in 8 distinct bank groups.
template <int RC>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  const int f = RC == 8 ? (row & 7) : ((row >> 1) & 3);
  return (uint32_t)(row * RC + (chunk ^ f)) * 16u;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ldsm4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void ldsm4t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {  // x ~ hi + lo, 22 bits
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(x - __uint_as_float(hi)));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
// 3xTF32: d += a_lo b_hi + a_hi b_lo + a_hi b_hi (b = {b0 hi, b1 hi, b0 lo, b1 lo})
__device__ __forceinline__ void mma3_tf32(float (&d)[4], const uint4& ah, const uint4& al, const uint4& b) {
  mma_tf32(d, al, b.x, b.y);
  mma_tf32(d, ah, b.z, b.w);
  mma_tf32(d, ah, b.x, b.y);
}
// fp16 split of a pair: hi = fp16(x), lo = fp16(x - hi) (paired conversions)
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x - hf.x, y - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// The power of two that puts m's leading bit at 2^14 (m in [2^14, 2^15) after
// scaling); 1 for m = 0 / inf / nan.  m = 1.f x 2^(E - 127) -> 2^(141 - E).
__device__ __forceinline__ float col_scale(float m) {
  if (!(m > 0.f) || !isfinite(m)) return 1.f;
  const int E = (__float_as_int(m) >> 23) & 0xff;  // 0 for subnormal m: clamped below
  const int f = 268 - E;
  return __int_as_float((f > 254 ? 254 : f) << 23);
}
template <int SEG>
__device__ __forceinline__ double seg_sum(double v) {  // sum over aligned SEG-lane segments
#pragma unroll
  for (int o = SEG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// q[rr] = sum_k G[i0 + rr][k] P[k][j]  (G, P row-major K x K complex in smem)
template <int K, int RG>
__device__ __forceinline__ void gemv_cols(const float2* Gs, const float2* Ps, int i0, int j, float2 (&qv)[RG]) {
#pragma unroll
  for (int rr = 0; rr < RG; ++rr) qv[rr] = make_float2(0.f, 0.f);
#pragma unroll 4
  for (int k = 0; k < K; k += 2) {
    const float2 p0 = Ps[k * K + j], p1 = Ps[(k + 1) * K + j];
#pragma unroll
    for (int rr = 0; rr < RG; ++rr) {
      const float4 a = *reinterpret_cast<const float4*>(Gs + (i0 + rr) * K + k);
      float2& q = qv[rr];
      q.x = fmaf(a.x, p0.x, q.x); q.x = fmaf(-a.y, p0.y, q.x);
      q.y = fmaf(a.x, p0.y, q.y); q.y = fmaf(a.y, p0.x, q.y);
      q.x = fmaf(a.z, p1.x, q.x); q.x = fmaf(-a.w, p1.y, q.x);
      q.y = fmaf(a.z, p1.y, q.y); q.y = fmaf(a.w, p1.x, q.y);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(NT, 2) small_k_kernel(Params p) {
  using g = G<K>;
  constexpr int NC = g::NC, RC = g::RC, NG = g::NG, US = g::US;
  extern __shared__ __align__(128) uint8_t smem[];
  const int M = p.M;
  uint8_t* Zh = smem;                                        // [M][NC] fp16, swizzled
  uint8_t* Zl = Zh + (size_t)M * NC * 2;
  float2* Gs = reinterpret_cast<float2*>(Zl + (size_t)M * NC * 2);  // [K][K] G = H^H H (no xi)
  float2* Ps = Gs + K * K;                                   // [K][K] P, then X
  uint8_t* XT = reinterpret_cast<uint8_t*>(Ps + K * K);      // Xe'^T hi | lo ([NC][NC] fp16) ...
  float* Us = reinterpret_cast<float*>(XT);                  // ... aliased by U ([NC][US] fp32)
  uint4* GA = reinterpret_cast<uint4*>(XT);                  // ... and by the K = 32 product A fragments
  uint4* BF = reinterpret_cast<uint4*>(Gs);                  // K = 32 product B fragments (over G, P)
  float* sc = reinterpret_cast<float*>(XT + g::XT_BYTES);    // [K] column scales s_k
  float* tcs = sc + K;                                       // [K] 1 / X' column scales t_j
  float* cdg = tcs + K;                                      // [K] A_ii
  float* isc = cdg + K;                                      // [K] 1 / s_k
  float* part1 = isc + K;                                    // [NG][K]
  float* part2 = part1 + NG * K;                             // [NG][K] (K = 32 SINR: [4][K] doubles)
  double* dred = reinterpret_cast<double*>(part2 + NG * K);  // [NW]
  float* sse = reinterpret_cast<float*>(dred + NW);          // [NW]
  int* flags = reinterpret_cast<int*>(sse + NW);             // [0] status bits, [1..K] column max bits
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  const bool alg1 = use_c && !textbook;
  const float xi = (float)(p.xi_b ? p.xi_b[b] : p.xi);

  // ---- H -> registers (16-B loads) -> per-user column max -> scaled fp16 split tiles
  {
    constexpr int PR = K / 2;  // float4 (two users) per antenna row
    constexpr int NLMAX = 8192 / (2 * NT);
    const float4* H4 = reinterpret_cast<const float4*>(p.H + b * (int64_t)M * K);
    const int nl = M * PR / NT;
    if (tid <= K) flags[tid] = 0;
    float4 v[NLMAX];
#pragma unroll
    for (int i = 0; i < NLMAX; ++i)
      if (i < nl) v[i] = __ldcs(H4 + tid + NT * i);
    const int u = tid % PR;  // this thread's user pair (2u, 2u + 1), fixed since NT % PR == 0
    float m0 = 0.f, m1 = 0.f;
#pragma unroll
    for (int i = 0; i < NLMAX; ++i)
      if (i < nl) {
        m0 = fmaxf(m0, fmaxf(fabsf(v[i].x), fabsf(v[i].y)));
        m1 = fmaxf(m1, fmaxf(fabsf(v[i].z), fabsf(v[i].w)));
      }
#pragma unroll
    for (int o = PR; o < 32; o <<= 1) {
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    __syncthreads();  // flags zeroed
    if (lane < PR) {
      atomicMax(&flags[1 + 2 * u], __float_as_int(m0));
      atomicMax(&flags[2 + 2 * u], __float_as_int(m1));
    }
    __syncthreads();
    const float s0 = col_scale(__int_as_float(flags[1 + 2 * u])), s1 = col_scale(__int_as_float(flags[2 + 2 * u]));
    if (tid < K) {
      const float sv = col_scale(__int_as_float(flags[1 + tid]));
      sc[tid] = sv;
      isc[tid] = 1.f / sv;  // exact: a power of two
    }
#pragma unroll
    for (int i = 0; i < NLMAX; ++i)
      if (i < nl) {
        const int a = (tid + NT * i) / PR;
        uint2 hi, lo;
        split2(v[i].x * s0, v[i].y * s0, hi.x, lo.x);
        split2(v[i].z * s1, v[i].w * s1, hi.y, lo.y);
        const uint32_t off = swz<RC>(a, u >> 1) + (u & 1) * 8;
        *reinterpret_cast<uint2*>(Zh + off) = hi;
        *reinterpret_cast<uint2*>(Zl + off) = lo;
      }
  }
  __syncthreads();

  // ---- Gram on the tensor cores: U = Zh^T Zh + 2 Zh^T Zl over the M antennas
  if (warp < g::GWARPS) {
    constexpr int GNP = g::GNP;
    const int m0 = (warp % g::MT) * 16, n0 = (warp / g::MT) * GNP * 8;
    float acc[GNP][4], acl[GNP][4];
#pragma unroll
    for (int n = 0; n < GNP; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[n][e] = acl[n][e] = 0.f;
    const int q = lane >> 3, r = lane & 7;
    const uint32_t zh = smem_u32(Zh), zl = smem_u32(Zl);
    for (int k0 = 0; k0 < M; k0 += 16) {
      uint32_t af[4];
      ldsm4t(zh + swz<RC>(k0 + r + (q >> 1) * 8, (m0 >> 3) + (q & 1)), af);  // A = Zh^T (m = comp, k = antenna)
#pragma unroll
      for (int n = 0; n < GNP; n += 2) {
        const uint32_t bo = swz<RC>(k0 + r + (q & 1) * 8, ((n0 + 8 * n) >> 3) + (q >> 1));
        uint32_t bh[4], bl[4];
        ldsm4t(zh + bo, bh);
        ldsm4t(zl + bo, bl);
        hmma(acc[n], af, bh[0], bh[1]);
        hmma(acc[n + 1], af, bh[2], bh[3]);
        hmma(acl[n], af, bl[0], bl[1]);
        hmma(acl[n + 1], af, bl[2], bl[3]);
      }
    }
    const int gr = lane >> 2, t2 = 2 * (lane & 3);
#pragma unroll
    for (int n = 0; n < GNP; ++n) {
      const int c = n0 + 8 * n + t2;
      *reinterpret_cast<float2*>(Us + (m0 + gr) * US + c) =
          make_float2(fmaf(2.f, acl[n][0], acc[n][0]), fmaf(2.f, acl[n][1], acc[n][1]));
      *reinterpret_cast<float2*>(Us + (m0 + gr + 8) * US + c) =
          make_float2(fmaf(2.f, acl[n][2], acc[n][2]), fmaf(2.f, acl[n][3], acc[n][3]));
    }
  }
  __syncthreads();

  // ---- G = H^H H (unscaled exactly; no xi: A p = G p + xi p)
  for (int e = tid; e < K * K; e += NT) {
    const int i = e / K, j = e % K;
    const float* u0 = Us + (2 * i) * US + 2 * j;
    const float* u1 = Us + (2 * i + 1) * US + 2 * j;
    const float* v0 = Us + (2 * j) * US + 2 * i;
    const float* v1 = Us + (2 * j + 1) * US + 2 * i;
    // sym(U)_cd = (U_cd + U_dc) / 2; Gr = sym(2i,2j) + sym(2i+1,2j+1); Gi = sym(2i,2j+1) - sym(2i+1,2j)
    const float s00 = 0.5f * (u0[0] + v0[0]), s11 = 0.5f * (u1[1] + v1[1]);
    const float s01 = 0.5f * (u0[1] + v1[0]), s10 = 0.5f * (u1[0] + v0[1]);
    const float inv = isc[i] * isc[j];  // exact: powers of two
    const float gr = (s00 + s11) * inv;
    Gs[i * K + j] = make_float2(gr, i == j ? 0.f : (s01 - s10) * inv);
    if (i == j) cdg[i] = gr + xi;  // A_ii: the Jacobi preconditioner
  }
  __syncthreads();

  // ---- element ownership: thread holds NE complex entries (ie[e], je[e]) of
  // X, R, P, Q, GX.  K = 32: the m16n8 accumulator layout of the tensor-core
  // products (warp = 16 rows x 8 columns); K = 16: row tid / 16, column tid % 16.
  constexpr int NE = K == 32 ? 4 : 1;
  const int gq = lane >> 2, tq = lane & 3, wmt = warp & 1, wnt = warp >> 1;
  int ie[NE], je[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    if constexpr (K == 32) {
      ie[e] = 16 * wmt + gq + 8 * (e >> 1);
      je[e] = 8 * wnt + 2 * tq + (e & 1);
    } else {
      ie[e] = tid / K;
      je[e] = tid % K;
    }
  }
  // column sums of one value per owned entry, in a fixed order (part: scratch [NG][K])
  constexpr int NCOLS = K == 32 ? 2 : 1;
  auto col_sums = [&](const float (&v)[NE], float* part, float (&out)[NCOLS], bool is_max) {
    if constexpr (K == 32) {
      float a = is_max ? fmaxf(v[0], v[2]) : v[0] + v[2];
      float c = is_max ? fmaxf(v[1], v[3]) : v[1] + v[3];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const float a2 = __shfl_xor_sync(0xffffffffu, a, o), c2 = __shfl_xor_sync(0xffffffffu, c, o);
        a = is_max ? fmaxf(a, a2) : a + a2;
        c = is_max ? fmaxf(c, c2) : c + c2;
      }
      if (gq == 0) {
        part[wmt * K + je[0]] = a;
        part[wmt * K + je[1]] = c;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float x0 = part[je[c]], x1 = part[K + je[c]];
        out[c] = is_max ? fmaxf(x0, x1) : x0 + x1;
      }
    } else {
      part[ie[0] * K + je[0]] = v[0];
      __syncthreads();
      float acc = part[je[0]];
#pragma unroll 4
      for (int gI = 1; gI < NG; ++gI) acc = is_max ? fmaxf(acc, part[gI * K + je[0]]) : acc + part[gI * K + je[0]];
      out[0] = acc;
    }
  };

  // P (or X) -> the operand of the next K x K product
  auto put_operand = [&](const float2 (&v)[NE]) {
    if constexpr (K == 32) {
      // B fragments of the 3xTF32 m16n8k8 products, [half re/im][ksub][column n][t] x {b0h, b1h, b0l, b1l}
      uint32_t* bw = reinterpret_cast<uint32_t*>(BF);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int k = ie[e], ksub = k >> 3, tt = k & 3, slot = (k >> 2) & 1;
        uint32_t h, l;
        split_tf32(v[e].x, h, l);
        uint32_t* w0 = bw + (((0 * 4 + ksub) * K + je[e]) * 4 + tt) * 4 + slot;
        w0[0] = h;
        w0[2] = l;
        split_tf32(v[e].y, h, l);
        uint32_t* w1 = bw + (((1 * 4 + ksub) * K + je[e]) * 4 + tt) * 4 + slot;
        w1[0] = h;
        w1[2] = l;
      }
    } else {
      Ps[ie[0] * K + je[0]] = v[0];
    }
  };
  // q = G v for the owned entries (v as last put_operand'ed)
  auto product = [&](float2 (&q)[NE]) {
    if constexpr (K == 32) {
      // eight independent accumulator chains (hi*hi apart from the two
      // correction terms; the Gr and Gi blocks apart) of <= 8 MMAs each
      float acc[8][4];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[a][e] = 0.f;
      const uint4* bre = BF + (0 * 4 * K + 8 * wnt + gq) * 4 + tq;
      const uint4* bim = BF + (1 * 4 * K + 8 * wnt + gq) * 4 + tq;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint4 ah = GA[((wmt * 8 + ks) * 32 + lane) * 2], al = GA[((wmt * 8 + ks) * 32 + lane) * 2 + 1];
        const uint4 br = bre[(ks & 3) * K * 4], bi = bim[(ks & 3) * K * 4];
        // Gr block (ks < 4): Qr += Gr Pr, Qi += Gr Pi; Gi block: Qr -= Gi Pi, Qi += Gi Pr
        const uint4& b1 = ks < 4 ? br : bi;
        const uint4& b2 = ks < 4 ? bi : br;
        const int o = ks < 4 ? 0 : 4;
        mma_tf32(acc[o + 0], ah, b1.x, b1.y);
        mma_tf32(acc[o + 1], al, b1.x, b1.y);
        mma_tf32(acc[o + 1], ah, b1.z, b1.w);
        mma_tf32(acc[o + 2], ah, b2.x, b2.y);
        mma_tf32(acc[o + 3], al, b2.x, b2.y);
        mma_tf32(acc[o + 3], ah, b2.z, b2.w);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        q[e] = make_float2((acc[0][e] + acc[1][e]) - (acc[4][e] + acc[5][e]),
                           (acc[2][e] + acc[3][e]) + (acc[6][e] + acc[7][e]));
    } else {
      gemv_cols<K, 1>(Gs, Ps, ie[0], je[0], q);
    }
  };

  if constexpr (K == 32) {
    // A fragments of the products: A = [Gr | Gi] (K x 2K), 3xTF32 split, per
    // [m-tile][k-step][lane] {a0..a3} hi then lo (in the U region, free now)
    for (int f = tid; f < 2 * 8 * 32; f += NT) {
      const int mt = f >> 8, ks = (f >> 5) & 7, ln = f & 31, g8 = ln >> 2, t8 = ln & 3;
      const int r0 = 16 * mt + g8, c0 = 8 * ks + t8;
      auto av = [&](int rr, int cc) { return cc < K ? Gs[rr * K + cc].x : Gs[rr * K + cc - K].y; };
      uint4 h, l;
      split_tf32(av(r0, c0), h.x, l.x);
      split_tf32(av(r0 + 8, c0), h.y, l.y);
      split_tf32(av(r0, c0 + 4), h.z, l.z);
      split_tf32(av(r0 + 8, c0 + 4), h.w, l.w);
      GA[2 * f] = h;
      GA[2 * f + 1] = l;
    }
  }

  // ---- Jac-PCG / CG (linsolve.py:217-294) on the K identity RHS, w0 = 0.
  // Per-column scalars (rz, alpha, beta) live in NCOL slots: entry e is in
  // column slot e % NCOL.
  constexpr int NCOL = K == 32 ? 2 : 1;
  float icr[NE], icc[NCOL], rz[NCOL];
  float2 x[NE], r[NE], pv[NE], qv[NE];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    icc[c] = use_c ? 1.f / cdg[je[c]] : 1.f;
    rz[c] = textbook ? icc[c] : (use_c ? icc[c] * icc[c] : 1.f);
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const float ci = cdg[ie[e]];
    icr[e] = use_c ? 1.f / ci : 1.f;
    if (use_c && ci == 0.f && ie[e] == je[e]) atomicOr(flags, 2);
    const float d = (ie[e] == je[e]) ? 1.f : 0.f;
    const float rv = alg1 ? d * icr[e] : d;
    x[e] = make_float2(0.f, 0.f);
    r[e] = make_float2(rv, 0.f);
    pv[e] = make_float2(textbook ? d * icr[e] : rv, 0.f);
    // first product: P0 = diag(p_jj), so (G + xi I) P0 is a column scaling
    // (every other term of the sum is an exact zero)
    const float pjj = use_c ? icc[e % NCOL] : 1.f;
    float2 gij = Gs[ie[e] * K + je[e]];
    if (ie[e] == je[e]) gij.x += xi;
    qv[e] = make_float2(gij.x * pjj, gij.y * pjj);
  }
  for (int t = 1; t <= p.T; ++t) {
    if (t > 1) {
      product(qv);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        qv[e].x = fmaf(xi, pv[e].x, qv[e].x);  // A p = G p + xi p
        qv[e].y = fmaf(xi, pv[e].y, qv[e].y);
      }
    }
    float cp[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const float qf = alg1 ? icr[e] : 1.f;  // Algorithm 1: z = C^-1 A p
      cp[e] = pv[e].x * (qv[e].x * qf) + pv[e].y * (qv[e].y * qf);
    }
    float curv[NCOL];
    col_sums(cp, part1, curv, false);
    float al[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const bool act = rz[c] > 0.f;
      if (curv[c] <= 0.f && act) atomicOr(flags, 1);
      al[c] = act ? rz[c] / (curv[c] > 0.f ? curv[c] : 1.f) : 0.f;
    }
    float rp[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const float a = al[e % NCOL], qf = alg1 ? icr[e] : 1.f;
      x[e].x = fmaf(a, pv[e].x, x[e].x);
      x[e].y = fmaf(a, pv[e].y, x[e].y);
      r[e].x -= a * (qv[e].x * qf);
      r[e].y -= a * (qv[e].y * qf);
      const float ic = textbook ? icr[e] : 1.f;
      rp[e] = r[e].x * (r[e].x * ic) + r[e].y * (r[e].y * ic);
    }
    if (t == p.T) break;  // the last direction update feeds nothing
    float rn[NCOL], be[NCOL];
    col_sums(rp, part2, rn, false);
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      be[c] = rz[c] > 0.f ? rn[c] / rz[c] : 0.f;
      rz[c] = rn[c];
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const float ic = textbook ? icr[e] : 1.f, bb = be[e % NCOL];
      pv[e] = make_float2(fmaf(r[e].x, ic, bb * pv[e].x), fmaf(r[e].y, ic, bb * pv[e].y));
    }
    // every thread is past this iteration's product (two barriers ago); at
    // t = 1 past the G reads of the fragment build and of the column scaling
    put_operand(pv);
    __syncthreads();
  }

  // ---- GX = G X; ||F||^2 = Re tr(X^H GX) (fp64); beta
  // (the loop left after the curvature barrier of iteration T: nothing reads the operand any more)
  put_operand(x);
  __syncthreads();
  float2 gx[NE];
  product(gx);
  double fp = 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) fp += (double)x[e].x * gx[e].x + (double)x[e].y * gx[e].y;
  fp = warp_sum(fp);
  if (lane == 0) dred[warp] = fp;
  // column max of X' = S^-1 X (the W operand scale t_j); the barrier inside
  // also publishes dred
  float xm[NE], cm[NCOLS];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const float is = isc[ie[e]];
    xm[e] = fmaxf(fabsf(x[e].x * is), fabsf(x[e].y * is));
  }
  col_sums(xm, part1, cm, true);
  double fro = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) fro += dred[w];
  const bool degenerate = !(fro > 0.0);
  const double btd = degenerate ? 0.0 : sqrt(p.power / fro);

  // Xe'^T (fp16 hi | lo): rows n = output components, columns c = input components
  {
    uint8_t* XTh = XT;
    uint8_t* XTl = XT + NC * NC * 2;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int i = ie[e], j = je[e];
      const float tj = col_scale(cm[e % NCOLS]);
      if (i == 0) tcs[j] = 1.f / tj;  // exact: a power of two
      const float f = tj * isc[i];
      const float xr = x[e].x * f, xim = x[e].y * f;
      uint32_t h0, l0, h1, l1;
      split2(xr, -xim, h0, l0);  // row 2j:     (Re, -Im) at columns 2i, 2i + 1
      split2(xim, xr, h1, l1);   // row 2j + 1: (Im,  Re)
      const int c = 2 * i;
      const uint32_t o0 = swz<RC>(2 * j, c >> 3) + (c & 7) * 2, o1 = swz<RC>(2 * j + 1, c >> 3) + (c & 7) * 2;
      *reinterpret_cast<uint32_t*>(XTh + o0) = h0;
      *reinterpret_cast<uint32_t*>(XTl + o0) = l0;
      *reinterpret_cast<uint32_t*>(XTh + o1) = h1;
      *reinterpret_cast<uint32_t*>(XTl + o1) = l1;
    }
  }
  if (p.X) {
    float2* Xo = p.X + b * (int64_t)K * K;
#pragma unroll
    for (int e = 0; e < NE; ++e) Xo[ie[e] * K + je[e]] = x[e];
  }

  // ---- SINR / SE from B = beta GX (row k: user k; interference summed directly)
  {
    const double b2 = btd * btd;
    double sig = 0.0, intf = 0.0;
    int diag_e = -1;
    if constexpr (K == 32) {
      // row partials over this thread's two columns, then over the 4 lanes of a row
      double rp2[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double v = b2 * ((double)gx[e].x * gx[e].x + (double)gx[e].y * gx[e].y);
        if (ie[e] == je[e]) {
          sig = v;
          diag_e = e;
        } else {
          rp2[e >> 1] += v;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        rp2[h] += __shfl_xor_sync(0xffffffffu, rp2[h], 1);
        rp2[h] += __shfl_xor_sync(0xffffffffu, rp2[h], 2);
      }
      double* rowp = reinterpret_cast<double*>(part2);  // [4 column groups][K]
      if (tq == 0) {
        rowp[wnt * K + ie[0]] = rp2[0];
        rowp[wnt * K + ie[2]] = rp2[1];
      }
      __syncthreads();
      if (diag_e >= 0) {
        const int i = ie[diag_e];
        intf = ((rowp[i] + rowp[K + i]) + rowp[2 * K + i]) + rowp[3 * K + i];
      }
    } else {
      const double v = b2 * ((double)gx[0].x * gx[0].x + (double)gx[0].y * gx[0].y);
      const bool d = ie[0] == je[0];
      intf = seg_sum<K>(d ? 0.0 : v);
      if (d) {
        sig = v;
        diag_e = 0;
      }
    }
    float se = 0.f;
    if (diag_e >= 0) {
      const double gam = sig / (intf + p.sigma2);
      if (p.gamma) p.gamma[b * K + ie[diag_e]] = gam;
      se = log1pf((float)gam) * 1.4426950408889634f;  // log2(1 + gamma)
    }
    se = warp_sum(se);
    if (lane == 0) sse[warp] = se;
  }
  __syncthreads();  // XT, tcs, sse

  // ---- W = beta Z' Xe' / t_j on the tensor cores (3xFP16), two m-tiles per warp step
  {
    constexpr int NTL = g::NTL;
    const uint32_t zh = smem_u32(Zh), zl = smem_u32(Zl), xh = smem_u32(XT), xl = xh + NC * NC * 2;
    const int q = lane >> 3, r8 = lane & 7, gr = lane >> 2, t4 = lane & 3;
    const float bt = (float)btd;
    float2* Wb = p.W + b * (int64_t)M * K;
    float2* Fb = p.F ? p.F + b * (int64_t)M * K : nullptr;
    float its[NTL];
#pragma unroll
    for (int n = 0; n < NTL; ++n) its[n] = tcs[4 * n + t4];
    for (int mp = warp; mp < M / 32; mp += NW) {
      float acc[2][NTL][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int n = 0; n < NTL; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[h][n][e] = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < NC; c0 += 16) {
        uint32_t ah[2][4], alo[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t ao = swz<RC>(32 * mp + 16 * h + r8 + (q & 1) * 8, (c0 >> 3) + (q >> 1));
          ldsm4(zh + ao, ah[h]);
          ldsm4(zl + ao, alo[h]);
        }
#pragma unroll
        for (int n = 0; n < NTL; n += 2) {
          const uint32_t bo = swz<RC>(8 * n + r8 + (q >> 1) * 8, (c0 >> 3) + (q & 1));
          uint32_t bh[4], bl[4];
          ldsm4(xh + bo, bh);
          ldsm4(xl + bo, bl);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            hmma(acc[h][n], ah[h], bh[0], bh[1]);
            hmma(acc[h][n], ah[h], bl[0], bl[1]);
            hmma(acc[h][n], alo[h], bh[0], bh[1]);
            hmma(acc[h][n + 1], ah[h], bh[2], bh[3]);
            hmma(acc[h][n + 1], ah[h], bl[2], bl[3]);
            hmma(acc[h][n + 1], alo[h], bh[2], bh[3]);
          }
        }
      }
#pragma unroll
      for (int n = 0; n < NTL; ++n) {
        const int ju = 4 * n + t4;  // user column of this thread's (re, im) pair
        const float it = its[n];
        const float ws = bt * it;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 32 * mp + 16 * h + gr;
          __stcs(Wb + (int64_t)a * K + ju, make_float2(acc[h][n][0] * ws, acc[h][n][1] * ws));
          __stcs(Wb + (int64_t)(a + 8) * K + ju, make_float2(acc[h][n][2] * ws, acc[h][n][3] * ws));
          if (Fb) {
            __stcs(Fb + (int64_t)a * K + ju, make_float2(acc[h][n][0] * it, acc[h][n][1] * it));
            __stcs(Fb + (int64_t)(a + 8) * K + ju, make_float2(acc[h][n][2] * it, acc[h][n][3] * it));
          }
        }
      }
    }
  }
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)sse[w];
    p.sum_se[b] = s;
    p.beta[b] = btd;
    int st = 0;
    if (flags[0] & 2) st = XL_STATUS_SPLITTING;
    else if (flags[0] & 1) st = XL_STATUS_NOT_HPD;
    else if (degenerate) st = XL_STATUS_DEGENERATE;
    p.status[b] = st;
  }
}

template <int K>
size_t smem_bytes(int M) {
  using g = G<K>;
  return (size_t)M * g::NC * 2 * 2 + 2 * (size_t)K * K * 8 + g::XT_BYTES + 4 * K * 4 + 2 * g::NG * K * 4 +
         NW * 8 + NW * 4 + (K + 1) * 4;
}

}  // namespace fs

bool fc64s_supported(int dtype, int method, int M, int K) {
  if (dtype != XL_C64 || (method != XL_JACPCG && method != XL_CG)) return false;
  const char* e = getenv("XL_SMALL_K_MMA");  // "0": keep the tcgen05 kernel (A/B, tests)
  if (e && e[0] == '0') return false;
  if (K != 16 && K != 32) return false;
  return M >= 32 && M % 32 == 0 && M * K <= 8192;
}

int fc64s_rzf(int method, int variant, const void* H, int64_t B, int M, int K, double xi, const double* xi_b,
              double power, int T, double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
              void* X, int32_t* status, cudaStream_t st) {
  fs::Params p{(const float2*)H, B, M, method, variant, T, xi, xi_b, power, sigma2, (float2*)W, (float2*)F,
               (float2*)X, beta, gamma, sum_se, status};
  if (K == 16) {
    const size_t sm = fs::smem_bytes<16>(M);
    cudaFuncSetAttribute(fs::small_k_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fs::small_k_kernel<16><<<(unsigned)B, fs::NT, sm, st>>>(p);
  } else {
    const size_t sm = fs::smem_bytes<32>(M);
    cudaFuncSetAttribute(fs::small_k_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fs::small_k_kernel<32><<<(unsigned)B, fs::NT, sm, st>>>(p);
  }
  return check_launch("fused c64 small K (mma.sync)");
}

}  // namespace xl
