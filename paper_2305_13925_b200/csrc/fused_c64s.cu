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
//   * The K x K solve on the same tensor cores in 3xTF32 (mma.sync m16n8k8;
//     TF32 keeps fp32's exponent range, so P and X need no scaling), the
//     vector recurrences in fp32 SIMT.  Warp w < K / 8 owns columns
//     [8w, 8w + 8) of X, R, P, Q (the RHS columns are independent) in the
//     products' accumulator layout: the column reductions are warp shuffles
//     and the B operand is the warp's own columns, so the PCG loop has no
//     block barrier.  G is kept without xi (A p = G p + xi p), so GX = G X
//     is an explicit product with no cancellation against xi X at low SNR;
//     P0 is diagonal (x0 = 0, b = I), so the first product is a column
//     scaling: T iterations cost T K x K products (GX included).
//
// Scaling: every user column k of Z (its re and im components) is scaled by
// s_k = 2^e_k so that its largest |component| lies in [2^14, 2^15) -- the
// fp16 split then keeps ~22 bits for every column regardless of the gain
// spread between users.  The Gram is unscaled exactly (A_ij = G'_ij / s_i s_j),
// and W uses Xe' = S^-1 X T with a per-output-column power of two t_j.
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
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
  int pf;  // L2 prefetch distance in realizations (the resident CTAs of the grid)
  long long* trace;  // dev (XL_SMALL_K_TRACE=<first CTA + 1>): clock64 phase stamps of 64 CTAs
  unsigned trace0;
};
#define STAMP(n)                                                               \
  do {                                                                         \
    if (p.trace && threadIdx.x == 0 && blockIdx.x - p.trace0 < 64u)                              \
      p.trace[(blockIdx.x - p.trace0) * 64 + (n)] = clock64();                                     \
  } while (0)

template <int K>
struct G {
  static constexpr int NC = 2 * K;        // real components (re/im interleaved, as in H)
  static constexpr int RC = NC * 2 / 16;  // 16-B chunks per fp16 row (8 for K = 32, 4 for K = 16)
  static constexpr int US = NC + 2;       // fp32 U row stride (2-way conflicts on the fragment stores)
  static constexpr int XT_BYTES = (NC * US * 4 > 2 * NC * NC * 2) ? NC * US * 4 : 2 * NC * NC * 2;
  static constexpr int MT = NC / 16, NTL = NC / 8;           // m16 / n8 tiles of a 2K x 2K product
  static constexpr int GNP = K == 32 ? 4 : 2;                // Gram n-tiles per warp
  static constexpr int GWARPS = MT * NTL / GNP;              // Gram warps (8 / 4)
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

template <int K>
__global__ void __launch_bounds__(NT, 2) small_k_kernel(Params p) {
  using g = G<K>;
  constexpr int NC = g::NC, RC = g::RC, US = g::US;
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
  double* rowp = reinterpret_cast<double*>(isc + K);         // [K / 8][K] SINR row partials
  double* dred = rowp + (K / 8) * K;                         // [NW]
  float* colx = reinterpret_cast<float*>(dred + NW);         // [3][K / 16][K] column exchange slots
  float* sse = colx + 3 * (K / 16) * K;                      // [NW]
  int* flags = reinterpret_cast<int*>(sse + NW);             // [0] status bits, [1..K] column max bits
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  const bool alg1 = use_c && !textbook;
  const float xi = (float)(p.xi_b ? p.xi_b[b] : p.xi);
  STAMP(0);

  // ---- H -> registers (16-B loads) -> per-user column max -> scaled fp16 split tiles
  {
    constexpr int PR = K / 2;  // float4 (two users) per antenna row
    constexpr int NLMAX = 8192 / (2 * NT);
    const float4* H4 = reinterpret_cast<const float4*>(p.H + b * (int64_t)M * K);
    const int nl = M * PR / NT;
    if (tid <= K) flags[tid] = 0;
    if (tid == 0 && b + p.pf < p.B) {  // the CTA that runs after the next wave finds its H in L2
      const float2* nx = p.H + (b + p.pf) * (int64_t)M * K;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx), "r"((uint32_t)(M * K * 8)) : "memory");
    }
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
    STAMP(1);
    if (lane < PR) {
      atomicMax(&flags[1 + 2 * u], __float_as_int(m0));
      atomicMax(&flags[2 + 2 * u], __float_as_int(m1));
    }
    __syncthreads();
    STAMP(2);
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
  STAMP(3);

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
  STAMP(4);

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
  STAMP(5);

  // ---- The solve.  Column block cb (8 RHS columns, independent of the
  // others) is owned by NMT = K / 16 warps, warp = one m16 row tile of it, in
  // the accumulator layout of its tensor-core products: entry e = 2 h + c is
  // (i = 16 mt + g + 8 h, j = 8 cb + 2 t + c).  Column reductions are warp
  // shuffles plus (K = 32) one exchange with the partner warp through shared
  // memory and a 64-thread named barrier; the B operand of a product is the
  // block's own columns.  No block-wide barrier inside the PCG loop.
  constexpr int NMT = K / 16, NCB = K / 8, NSW = NMT * NCB, KS = K / 4, KSUB = K / 8, NE = 4;
  static_assert(NSW <= NW, "solver warps");
  const int gq = lane >> 2, tq = lane & 3;
  const int cb = warp / NMT, mt = warp % NMT;
  const bool solver = warp < NSW;
  // A fragments of the products: A = [Gr | Gi] (K x 2K), 3xTF32 split, per
  // [m-tile][k-step][lane] {a0..a3} hi then lo (in the U region, free now)
  for (int f = tid; f < NMT * KS * 32; f += NT) {
    const int fm = f / (KS * 32), ks = (f / 32) % KS, ln = f & 31, g8 = ln >> 2, t8 = ln & 3;
    const int r0 = 16 * fm + g8, c0 = 8 * ks + t8;
    auto av = [&](int rr, int cc) { return cc < K ? Gs[rr * K + cc].x : Gs[rr * K + cc - K].y; };
    uint4 h, l;
    split_tf32(av(r0, c0), h.x, l.x);
    split_tf32(av(r0 + 8, c0), h.y, l.y);
    split_tf32(av(r0, c0 + 4), h.z, l.z);
    split_tf32(av(r0 + 8, c0 + 4), h.w, l.w);
    GA[2 * f] = h;
    GA[2 * f + 1] = l;
  }
  int ie[NE], je[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    ie[e] = 16 * mt + gq + 8 * (e >> 1);
    je[e] = 8 * cb + 2 * tq + (e & 1);
  }
  auto pair_sync = [&]() {  // the NMT warps of column block cb (immediate barrier ids 1..NCB)
    if constexpr (NMT > 1) {
      switch (cb) {
        case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
        case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
        case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
        default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
      }
    } else {
      __syncwarp();
    }
  };
  static_assert(NMT <= 2 && NCB <= 4, "pair barriers");
  // column c in {0, 1} of this thread: its two rows, the 8 row lanes, then the
  // partner warp's half through exchange slot `slot` (fixed order: mt 0 + mt 1)
  auto col_sum = [&](const float (&v)[NE], float (&out)[2], bool is_max, int slot) {
    float a[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      a[c] = is_max ? fmaxf(v[c], v[2 + c]) : v[c] + v[2 + c];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const float a2 = __shfl_xor_sync(0xffffffffu, a[c], o);
        a[c] = is_max ? fmaxf(a[c], a2) : a[c] + a2;
      }
    }
    if constexpr (NMT > 1) {
      float* xs = colx + slot * (NMT * K);  // [slot][mt][j]
      if (gq == 0) {
        xs[mt * K + je[0]] = a[0];
        xs[mt * K + je[1]] = a[1];
      }
      pair_sync();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float x0 = xs[je[c]], x1 = xs[K + je[c]];
        out[c] = is_max ? fmaxf(x0, x1) : x0 + x1;
      }
    } else {
      out[0] = a[0];
      out[1] = a[1];
    }
  };
  // v (P or X: this warp's rows of its block's columns) -> B fragments
  // [half re/im][ksub][column n][t] x {b0h, b1h, b0l, b1l}; then the pair barrier
  auto put_operand = [&](const float2 (&v)[NE]) {
    uint32_t* bw = reinterpret_cast<uint32_t*>(BF);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int k = ie[e], ksub = k >> 3, tt = k & 3, slot = (k >> 2) & 1;
      uint32_t h, l;
      split_tf32(v[e].x, h, l);
      uint32_t* w0 = bw + (((0 * KSUB + ksub) * K + je[e]) * 4 + tt) * 4 + slot;
      w0[0] = h;
      w0[2] = l;
      split_tf32(v[e].y, h, l);
      uint32_t* w1 = bw + (((1 * KSUB + ksub) * K + je[e]) * 4 + tt) * 4 + slot;
      w1[0] = h;
      w1[2] = l;
    }
    pair_sync();
  };
  // q = G v on this warp's tile (v as last put_operand'ed): Qr = Gr Vr - Gi Vi,
  // Qi = Gr Vi + Gi Vr; four accumulator chains (hi*hi apart from the two
  // correction terms) of KS and 2 KS MMAs
  auto product = [&](float2 (&q)[NE]) {
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int d = 0; d < 4; ++d) acc[a][d] = 0.f;
    const uint4* bre = BF + (0 * KSUB * K + 8 * cb + gq) * 4 + tq;
    const uint4* bim = BF + (1 * KSUB * K + 8 * cb + gq) * 4 + tq;
    const uint4* ga = GA + (mt * KS * 32 + lane) * 2;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint4 br = bre[(ks % KSUB) * K * 4], bi = bim[(ks % KSUB) * K * 4];
      const uint4 ah = ga[ks * 64], al = ga[ks * 64 + 1];
      uint4 b1 = br, b2 = bi;  // Gr block: Qr += Gr Vr, Qi += Gr Vi
      if (ks >= KSUB) {        // Gi block: Qr += Gi (-Vi), Qi += Gi Vr
        b1 = make_uint4(bi.x ^ 0x80000000u, bi.y ^ 0x80000000u, bi.z ^ 0x80000000u, bi.w ^ 0x80000000u);
        b2 = br;
      }
      mma_tf32(acc[0], ah, b1.x, b1.y);
      mma_tf32(acc[1], al, b1.x, b1.y);
      mma_tf32(acc[1], ah, b1.z, b1.w);
      mma_tf32(acc[2], ah, b2.x, b2.y);
      mma_tf32(acc[3], al, b2.x, b2.y);
      mma_tf32(acc[3], ah, b2.z, b2.w);
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) q[d] = make_float2(acc[0][d] + acc[1][d], acc[2][d] + acc[3][d]);
  };

  // ---- Jac-PCG / CG (linsolve.py:217-294) on the K identity RHS, w0 = 0
  float icr[NE], icc[2], rz[2];
  float2 x[NE], r[NE], pv[NE], qv[NE];
  if (solver) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
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
      const float pjj = use_c ? icc[e & 1] : 1.f;
      float2 gij = Gs[ie[e] * K + je[e]];
      if (ie[e] == je[e]) gij.x += xi;
      qv[e] = make_float2(gij.x * pjj, gij.y * pjj);
    }
  }
  __syncthreads();  // G read (fragments, first product): the operand region may overwrite it
  STAMP(11);
  if (solver) {
    for (int t = 1; t <= p.T; ++t) {
      if (t > 1) {
        product(qv);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          qv[e].x = fmaf(xi, pv[e].x, qv[e].x);  // A p = G p + xi p
          qv[e].y = fmaf(xi, pv[e].y, qv[e].y);
        }
      }
      STAMP(12 + 4 * t);
      float cp[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const float qf = alg1 ? icr[e] : 1.f;  // Algorithm 1: z = C^-1 A p
        cp[e] = pv[e].x * (qv[e].x * qf) + pv[e].y * (qv[e].y * qf);
      }
      float curv[2], al[2];
      col_sum(cp, curv, false, 0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool act = rz[c] > 0.f;
        if (curv[c] <= 0.f && act) atomicOr(flags, 1);
        al[c] = act ? rz[c] / (curv[c] > 0.f ? curv[c] : 1.f) : 0.f;
      }
      float rp[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const float a = al[e & 1], qf = alg1 ? icr[e] : 1.f;
        x[e].x = fmaf(a, pv[e].x, x[e].x);
        x[e].y = fmaf(a, pv[e].y, x[e].y);
        r[e].x -= a * (qv[e].x * qf);
        r[e].y -= a * (qv[e].y * qf);
        const float ic = textbook ? icr[e] : 1.f;
        rp[e] = r[e].x * (r[e].x * ic) + r[e].y * (r[e].y * ic);
      }
      if (t == p.T) break;  // the last direction update feeds nothing
      STAMP(13 + 4 * t);
      float rn[2], be[2];
      col_sum(rp, rn, false, 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        be[c] = rz[c] > 0.f ? rn[c] / rz[c] : 0.f;
        rz[c] = rn[c];
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const float ic = textbook ? icr[e] : 1.f, bb = be[e & 1];
        pv[e] = make_float2(fmaf(r[e].x, ic, bb * pv[e].x), fmaf(r[e].y, ic, bb * pv[e].y));
      }
      STAMP(14 + 4 * t);
      put_operand(pv);  // the partner is past this iteration's product (barrier of slot 0)
      STAMP(15 + 4 * t);
    }
  }
  STAMP(6);

  // ---- GX = G X (own tile); ||F||^2 = Re tr(X^H GX) (fp64); SINR row partials
  float2 gx[NE];
  double sig = 0.0;
  int diag_i = -1;
  if (solver) {
    put_operand(x);  // the partner is past its last product (barrier of slot 0 in iteration T)
    product(gx);
    double fp = 0.0;
#pragma unroll
    for (int e = 0; e < NE; ++e) fp += (double)x[e].x * gx[e].x + (double)x[e].y * gx[e].y;
    fp = warp_sum(fp);
    if (lane == 0) dred[warp] = fp;
    // row partials of |GX|^2 over this block's 8 columns (the diagonal apart)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      double v2 = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int e = 2 * hh + c;
        const double v = (double)gx[e].x * gx[e].x + (double)gx[e].y * gx[e].y;
        if (ie[e] == je[e]) {
          sig = v;
          diag_i = ie[e];
        } else {
          v2 += v;
        }
      }
      v2 += __shfl_xor_sync(0xffffffffu, v2, 1);
      v2 += __shfl_xor_sync(0xffffffffu, v2, 2);
      if (tq == 0) rowp[cb * K + ie[2 * hh]] = v2;
    }
    // column max of X' = S^-1 X (the W operand scale t_j): this warp's rows,
    // combined with the partner's after the block barrier
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float a = fmaxf(fmaxf(fabsf(x[c].x), fabsf(x[c].y)) * isc[ie[c]],
                      fmaxf(fabsf(x[2 + c].x), fabsf(x[2 + c].y)) * isc[ie[2 + c]]);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
      if (gq == 0) colx[2 * NMT * K + mt * K + je[c]] = a;
    }
  }
  __syncthreads();
  STAMP(8);
  double fro = 0.0;
#pragma unroll
  for (int w = 0; w < NSW; ++w) fro += dred[w];
  const bool degenerate = !(fro > 0.0);
  const double btd = degenerate ? 0.0 : sqrt(p.power / fro);

  if (solver) {
    // SINR / SE from B = beta GX (row k: user k; interference summed directly)
    float se = 0.f;
    if (diag_i >= 0) {
      const int i = diag_i;
      double intf = 0.0;
#pragma unroll
      for (int w = 0; w < NCB; ++w) intf += rowp[w * K + i];
      const double b2 = btd * btd;
      const double gam = (b2 * sig) / (b2 * intf + p.sigma2);
      if (p.gamma) p.gamma[b * K + i] = gam;
      se = log1pf((float)gam) * 1.4426950408889634f;  // log2(1 + gamma)
    }
    se = warp_sum(se);
    if (lane == 0) sse[warp] = se;
    // Xe'^T (fp16 hi | lo): rows n = output components, columns c = input components
    uint8_t* XTh = XT;
    uint8_t* XTl = XT + NC * NC * 2;
    float tjc[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float m = colx[2 * NMT * K + je[c]];
#pragma unroll
      for (int q2 = 1; q2 < NMT; ++q2) m = fmaxf(m, colx[2 * NMT * K + q2 * K + je[c]]);
      tjc[c] = col_scale(m);
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int i = ie[e], j = je[e];
      const float tj = tjc[e & 1];
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
    if (p.X) {
      float2* Xo = p.X + b * (int64_t)K * K;
#pragma unroll
      for (int e = 0; e < NE; ++e) Xo[ie[e] * K + je[e]] = x[e];
    }
  }
  __syncthreads();  // XT, tcs, sse
  STAMP(10);

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
      STAMP(7);
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
  STAMP(9);
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < (K / 16) * (K / 8); ++w) s += (double)sse[w];
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
  return (size_t)M * g::NC * 2 * 2 + 2 * (size_t)K * K * 8 + g::XT_BYTES + 4 * K * 4 + (K / 8) * K * 8 +
         NW * 8 + 3 * (K / 16) * K * 4 + NW * 4 + (K + 1) * 4;
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
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  fs::Params p{(const float2*)H, B, M, method, variant, T, xi, xi_b, power, sigma2, (float2*)W, (float2*)F,
               (float2*)X, beta, gamma, sum_se, status, 0, nullptr, 0};
  static long long* trace = nullptr;
  const char* tr = getenv("XL_SMALL_K_TRACE");
  if (tr && atoi(tr) > 0) {
    p.trace0 = (unsigned)(atoi(tr) - 1);
    if (!trace) cudaMalloc(&trace, 64 * 64 * sizeof(long long));
    cudaMemsetAsync(trace, 0, 64 * 64 * sizeof(long long), st);
    p.trace = trace;
  }
  auto launch = [&](auto kern, size_t sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fs::NT, sm);
    p.pf = (per_sm > 0 ? per_sm : 1) * nsm;
    kern<<<(unsigned)B, fs::NT, sm, st>>>(p);
  };
  if (K == 16) launch(fs::small_k_kernel<16>, fs::smem_bytes<16>(M));
  else launch(fs::small_k_kernel<32>, fs::smem_bytes<32>(M));
  if (p.trace) {  // dev: per-phase cycle deltas, averaged over the traced CTAs
    static long long h[64 * 64];
    cudaMemcpyAsync(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double acc[64] = {0};
    int n = 0;
    for (int c = 0; c < 64 && c + (int64_t)p.trace0 < B; ++c, ++n)
      for (int k = 1; k < 64; ++k)
        if (h[c * 64 + k]) acc[k] += (double)(h[c * 64 + k] - h[c * 64]);
    fprintf(stderr, "small_k trace (cycles since start, mean of %d CTAs):", n);
    for (int k = 1; k < 64; ++k)
      if (acc[k] != 0) fprintf(stderr, " %d:%.0f", k, acc[k] / n);
    fprintf(stderr, "\n");
  }
  return check_launch("fused c64 small K (mma.sync)");
}

}  // namespace xl
