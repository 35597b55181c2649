// Fused complex64 precoder for small K (K in {16, 32}) with the realization's
// H resident in shared memory: one CTA per realization, two CTAs per SM.
//
//   A = H^H H + xi I        gram_regularized (precoder.py:53-61)
//   Jac-PCG / CG, T iters   linsolve.py:217-294 on the K identity RHS, w0 = 0
//   or direct: X = A^-1     rzf_direct (precoder.py:73-78), Gauss-Jordan in place
//   GX, ||F||^2, beta       precoder.py:64-70 (K x K form)
//   W = beta H X, F = H X   precoder.py:90
//   B = beta GX, SINR, SE   coupling + sinr_eq9 (metrics.py:35-58)
//
// Why a separate kernel.  At K <= 32 the persistent tcgen05 kernel
// (fused_tc.cu) is bound by its math role's latency chain (one realization
// per SM at a time, a TMEM round trip and seven barrier rounds per PCG
// iteration).  Here two realizations share an SM and the
// work is split by the unit that suits it:
//
//   * Gram and W (the M x 2K x 2K products, ~90% of the flops), 3xFP16 like
//     fused_tc.cu: x = hi + lo, hi = fp16(x), lo = fp16(x - hi);
//     W = Zh Xh + Zh Xl + Zl Xh, and the Gram as U = Zh^T Zh + 2 Zh^T Zl,
//     G = (U + U^T) / 2 (Hermitian by construction).  TC (K = 32, M % 128
//     == 0): tcgen05 with TMEM accumulators -- the XOR-swizzled tiles are the
//     SWIZZLE_128B canonical layout -- and W leaving through SWIZZLE_128B
//     staging + 2-D TMA tensor stores; otherwise mma.sync m16n8k16 from the
//     same tiles through ldmatrix.
//   * The K x K solve's products on mma.sync in 3xFP16 on G' = D G D and
//     B' = D^-1 P F (D, F powers of two: D from G's diagonal, F from a
//     per-column bound on P's largest component), A fragments held in
//     registers for the whole solve; the vector recurrences in fp32 SIMT.
//     Column block cb (8 RHS columns; the columns are independent) is owned
//     by K / 16 warps in the products' accumulator layout: the column
//     reductions are warp shuffles plus one pair exchange, and the B operand
//     is the block's own columns, so the PCG loop has no block barrier.  G is
//     kept without xi (A p = G p + xi p), so GX = G X is an explicit product
//     with no cancellation against xi X at low SNR; P0 is diagonal (x0 = 0,
//     b = I), so the first product is a column scaling: T iterations cost T
//     K x K products (GX included).
//
// Scaling: every user column k of Z (its re and im components) is scaled by
// s_k = 2^e_k so that its largest |component| lies in [2^14, 2^15) -- the
// fp16 split then keeps ~22 bits for every column regardless of the gain
// spread between users.  The Gram is unscaled exactly (A_ij = G'_ij / s_i s_j),
// and W uses Xe' = S^-1 X T with a per-output-column power of two t_j.
#include <cuda.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "xl_common.cuh"

namespace xl {
namespace fs {
namespace t {
#include "tc_ptx.cuh"  // tcgen05 / TMEM / mbarrier wrappers (TC variant)
}

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
  static constexpr int GNP = 2;                              // Gram n-tiles per warp
  static constexpr int GMP = K == 32 ? 2 : 1;                // Gram m-tiles per warp
  static constexpr int GWARPS = MT * NTL / (GNP * GMP);      // Gram warps (8 / 4)
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
// fp16 split of a pair: hi = fp16(x), lo = fp16(x - hi) (paired conversions)
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const float2 v = make_float2(x, y);
  const __half2 h = __float22half2_rn(v);
  const float2 hf = __half22float2(h);
  const __half2 l = __float22half2_rn(__fadd2_rn(v, make_float2(-hf.x, -hf.y)));
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// The power of two s with m s in [2^(t-1), 2^t); 1 for m = 0 / inf / nan.
// m = 1.f x 2^(E - 127) -> s = 2^(t - 1 - (E - 127)), biased exponent t + 253 - E.
template <int TB>
__device__ __forceinline__ float pow2s(float m) {
  if (!(m > 0.f) || !isfinite(m)) return 1.f;
  const int E = (__float_as_int(m) >> 23) & 0xff;  // 0 for subnormal m: clamped below
  const int f = TB + 253 - E;
  return __int_as_float((f > 254 ? 254 : (f < 1 ? 1 : f)) << 23);
}
// 1 / s for a power of two s in the normal range (exact)
// 1 / v by rcp.approx and one Newton step: within an ulp or two of the rounded
// quotient, and without the range-check branch of the IEEE reciprocal (those
// branches sit on the latency-bound solver chains)
__device__ __forceinline__ float rcp_nr(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r * fmaf(-v, r, 2.f);
}
__device__ __forceinline__ float pow2_inv(float s) {
  return __int_as_float((254 - ((__float_as_int(s) >> 23) & 0xff)) << 23);
}
// the per-column scale of the fp16 W / Gram operands: max in [2^14, 2^15)
__device__ __forceinline__ float col_scale(float m) { return pow2s<15>(m); }
// tcgen05.ld 16x256b x8: 16 TMEM lanes x 64 columns; thread t gets, per 8-column
// group n, (lane t/4, cols 8n + 2(t%4), +1) then (lane t/4 + 8, same columns)
__device__ __forceinline__ void tmem_ld_16x256b_x8(uint32_t ta, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// tcgen05 shared-memory descriptor, SWIZZLE_128B (layout type 2 at bits 61-63,
// version 1 at bit 46; addresses and offsets in 16-B units)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
template <int SEG>
__device__ __forceinline__ double seg_sum(double v) {  // sum over aligned SEG-lane segments
#pragma unroll
  for (int o = SEG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// TC (K = 32, M % 128 == 0): the Gram and W run on tcgen05 (TMEM accumulators,
// one elected lane issues, async), Z and Xe' in the canonical no-swizzle
// core-matrix layout, the W epilogue from TMEM (thread = antenna row).
// Otherwise both run on mma.sync from XOR-swizzled tiles.
template <int K, bool TC>
__global__ void __launch_bounds__(NT, 2) small_k_kernel(Params p, const __grid_constant__ CUtensorMap wmap) {
  using g = G<K>;
  constexpr int NC = g::NC, RC = g::RC, US = g::US;
  static_assert(!TC || K == 32, "tcgen05 variant: K = 32");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int M = p.M;
  uint8_t* Zh = smem;                                        // [M][NC] fp16, swizzled (= SWIZZLE_128B canonical)
  uint8_t* Zl = Zh + (size_t)M * NC * 2;
  float2* Gs = reinterpret_cast<float2*>(Zl + (size_t)M * NC * 2);  // [K][K] G = H^H H (no xi)
  float2* Ps = Gs + K * K;                                   // [K][K] P, then X
  uint8_t* XT = reinterpret_cast<uint8_t*>(Ps + K * K);      // Xe'^T hi | lo ([NC][NC] fp16) ...
  float* Us = reinterpret_cast<float*>(XT);                  // ... aliased by U ([NC][US] fp32)
  uint4* BF = reinterpret_cast<uint4*>(Gs);                  // K x K product B' fragments (over G, P)
  float* sc = reinterpret_cast<float*>(XT + g::XT_BYTES);    // [K] column scales s_k
  float* tcs = sc + K;                                       // [K] 1 / X' column scales t_j
  float* cdg = tcs + K;                                      // [K] A_ii
  float* isc = cdg + K;                                      // [K] 1 / s_k
  float* dsc = isc + K;                                      // [K] G' = D G D row / column scales
  float* idsc = dsc + K;                                     // [K] 1 / dsc
  double* rowp = reinterpret_cast<double*>(idsc + K);        // [K / 8][K] SINR row partials
  double* dred = rowp + (K / 8) * K;                         // [NW]
  float* colx = reinterpret_cast<float*>(dred + NW);         // [5][K / 16][K] column exchange slots
  float* sse = colx + 5 * (K / 16) * K;                      // [NW]
  int* flags = reinterpret_cast<int*>(sse + NW);             // [0] status bits, [1..K] column max bits
  uint64_t* mbar = reinterpret_cast<uint64_t*>(flags + ((K + 2) & ~1));  // TC: MMA completion
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);             // TC: TMEM base
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  const bool alg1 = use_c && !textbook;
  const bool direct = p.method == XL_DIRECT;
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
    if constexpr (TC) {
      if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      }
      if (tid == 0) {
        t::mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
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
    if constexpr (TC) t::tc_before();
    __syncthreads();  // flags zeroed (TC: TMEM allocated, barrier initialised)
    if constexpr (TC) t::tc_after();
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
      isc[tid] = pow2_inv(sv);
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
  if constexpr (TC) t::fence_async_smem();  // generic-proxy tile writes -> the tensor cores' async proxy
  __syncthreads();
  STAMP(3);
  const uint32_t tmem = TC ? *tslot : 0u;

  // ---- Gram on the tensor cores: U = Zh^T Zh + 2 Zh^T Zl over the M antennas
  // (warp tile GMP m16 x GNP n8: the A and B fragment loads per k-step are
  // balanced, 4 ldmatrix.x4 per warp at K = 32)
  if constexpr (TC) {
    // U (TMEM cols 0-63) = Zh^T Zh, V (cols 64-127) = Zh^T Zl: M = 128 (the second
    // 64-component atom of A is the Zl plane: rows 64-127 ignored), N = 64, K = 16
    // antennas per MMA.  The swizzled tiles are SWIZZLE_128B canonical (MN-major
    // here: a 128-B row holds one antenna's 64 components)
    constexpr uint32_t IDG = t::idesc(128, NC, 1, 1);
    constexpr uint32_t ZPL = 256 * NC * 2;  // one 256-antenna fp16 plane
    if (warp == 0) {
      t::tc_after();
      const uint32_t zh = smem_u32(Zh), zl = smem_u32(Zl);
      if ((zh & 1023u) != 0) asm volatile("trap;");  // SWIZZLE_128B atoms need 1024-B alignment
      for (int ks = 0; ks < M / 16; ++ks) {
        const uint64_t dh = sw128_desc(zh + ks * 2048, ZPL, 1024), dl = sw128_desc(zl + ks * 2048, ZPL, 1024);
        t::mma_w(tmem, dh, dh, IDG, ks > 0);
        t::mma_w(tmem + 64, dh, dl, IDG, ks > 0);
      }
      t::commit_w(mbar);
    }
    t::mbar_wait(mbar, 0);
    t::tc_after();
    if ((warp & 3) < 2) {  // TMEM lanes 0-63 = U rows (component c1); warps 0, 1 | 4, 5: column halves
      const int c0 = 32 * (warp >> 2);
      float d[32], e2[32];
      t::tmem_ld<32>(tmem + ((32u * (warp & 3)) << 16) + c0, d);
      t::tmem_ld<32>(tmem + ((32u * (warp & 3)) << 16) + 64 + c0, e2);
      t::tmem_wait_ld();
      float* ur = Us + (32 * (warp & 3) + lane) * US + c0;
#pragma unroll
      for (int c = 0; c < 32; c += 2)
        *reinterpret_cast<float2*>(ur + c) = make_float2(fmaf(2.f, e2[c], d[c]), fmaf(2.f, e2[c + 1], d[c + 1]));
    }
  } else if (warp < g::GWARPS) {
    constexpr int GNP = g::GNP, GMP = g::GMP;
    const int m0 = (warp % (g::MT / GMP)) * 16 * GMP, n0 = (warp / (g::MT / GMP)) * GNP * 8;
    float acc[GMP][GNP][4], acl[GMP][GNP][4];
#pragma unroll
    for (int mm = 0; mm < GMP; ++mm)
#pragma unroll
      for (int n = 0; n < GNP; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[mm][n][e] = acl[mm][n][e] = 0.f;
    const int q = lane >> 3, r = lane & 7;
    const uint32_t zh = smem_u32(Zh), zl = smem_u32(Zl);
    for (int k0 = 0; k0 < M; k0 += 16) {
      uint32_t af[GMP][4];
#pragma unroll
      for (int mm = 0; mm < GMP; ++mm)  // A = Zh^T (m = comp, k = antenna)
        ldsm4t(zh + swz<RC>(k0 + r + (q >> 1) * 8, ((m0 + 16 * mm) >> 3) + (q & 1)), af[mm]);
#pragma unroll
      for (int n = 0; n < GNP; n += 2) {
        const uint32_t bo = swz<RC>(k0 + r + (q & 1) * 8, ((n0 + 8 * n) >> 3) + (q >> 1));
        uint32_t bh[4], bl[4];
        ldsm4t(zh + bo, bh);
        ldsm4t(zl + bo, bl);
#pragma unroll
        for (int mm = 0; mm < GMP; ++mm) {
          hmma(acc[mm][n], af[mm], bh[0], bh[1]);
          hmma(acc[mm][n + 1], af[mm], bh[2], bh[3]);
          hmma(acl[mm][n], af[mm], bl[0], bl[1]);
          hmma(acl[mm][n + 1], af[mm], bl[2], bl[3]);
        }
      }
    }
    const int gr = lane >> 2, t2 = 2 * (lane & 3);
#pragma unroll
    for (int mm = 0; mm < GMP; ++mm)
#pragma unroll
      for (int n = 0; n < GNP; ++n) {
        const int c = n0 + 8 * n + t2, rr = m0 + 16 * mm + gr;
        *reinterpret_cast<float2*>(Us + rr * US + c) =
            make_float2(fmaf(2.f, acl[mm][n][0], acc[mm][n][0]), fmaf(2.f, acl[mm][n][1], acc[mm][n][1]));
        *reinterpret_cast<float2*>(Us + (rr + 8) * US + c) =
            make_float2(fmaf(2.f, acl[mm][n][2], acc[mm][n][2]), fmaf(2.f, acl[mm][n][3], acc[mm][n][3]));
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
    if (i == j) {
      cdg[i] = gr + xi;  // A_ii: the Jacobi preconditioner
      // D: sqrt(G_ii) d_i in [2^6, 2^7), so |G'_ij| <= sqrt(G'_ii G'_jj) < 2^14 (fp16 range)
      const float d = pow2s<7>(sqrtf(gr));
      dsc[i] = d;
      idsc[i] = pow2_inv(d);
    }
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
  constexpr int NMT = K / 16, NCB = K / 8, NSW = NMT * NCB, KS = K / 8, KSUB = K / 16, NE = 4;
  static_assert(NSW <= NW, "solver warps");
  const int gq = lane >> 2, tq = lane & 3;
  const int cb = warp / NMT, mt = warp % NMT;
  const bool solver = warp < NSW;
  // The K x K products run on mma.sync m16n8k16 in 3xFP16 on G' = D G D
  // (D = diag(d_i), powers of two) and B' = D^-1 V F (F = diag(f_j), powers
  // of two from a bound on each column's largest component): q = G v =
  // D^-1 (G' B') F^-1, every scaling exact.  A = [G'r | G'i] (K x 2K): this
  // warp's m-tile fragments (hi, lo) stay in registers for the whole solve.
  uint32_t afh[KS][4], afl[KS][4];
  if (solver) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int rg = 0; rg < 4; ++rg) {
        const int i = 16 * mt + gq + 8 * (rg & 1), c = 16 * ks + 2 * tq + 8 * (rg >> 1);
        const int k = c < K ? c : c - K;  // the pair (c, c + 1) lies in one half
        const float2 g0 = Gs[i * K + k], g1 = Gs[i * K + k + 1];
        const float di = dsc[i];
        const float v0 = (c < K ? g0.x : g0.y) * di * dsc[k], v1 = (c < K ? g1.x : g1.y) * di * dsc[k + 1];
        split2(v0, v1, afh[ks][rg], afl[ks][rg]);
      }
  }
  int ie[NE], je[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    ie[e] = 16 * mt + gq + 8 * (e >> 1);
    je[e] = 8 * cb + 2 * tq + (e & 1);
  }
  auto pair_sync = [&]() {  // the NMT warps of column block cb (immediate barrier ids 1..NCB)
    if constexpr (NMT > 1) {
      asm volatile("bar.sync %0, 64;" ::"r"(cb + 1) : "memory");  // warp-uniform id, no branch
    } else {
      __syncwarp();
    }
  };
  static_assert(NMT <= 2 && NCB <= 4, "pair barriers");
  // column c in {0, 1} of this thread: its two rows, the 8 row lanes, then the
  // partner warp's half through exchange slot `slot` (fixed order: mt 0 + mt 1)
  auto col_red = [&](float a0, float a1, bool is_max, int slot, float (&out)[2], bool sync) {
    float a[2] = {a0, a1};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const float a2 = __shfl_xor_sync(0xffffffffu, a[c], o);
        a[c] = is_max ? fmaxf(a[c], a2) : a[c] + a2;
      }
    if constexpr (NMT > 1) {
      float* xs = colx + slot * (NMT * K);  // [slot][mt][j]
      if (gq == 0) {
        xs[mt * K + je[0]] = a[0];
        xs[mt * K + je[1]] = a[1];
      }
      if (sync) pair_sync();
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
  auto col_sum = [&](const float (&v)[NE], float (&out)[2], bool is_max, int slot) {
    col_red(is_max ? fmaxf(v[0], v[2]) : v[0] + v[2], is_max ? fmaxf(v[1], v[3]) : v[1] + v[3], is_max, slot, out,
            true);
  };
  // B' fragments [half re/im][ksub][column n][slot t ^ ((n >> 1) & 3)] x
  // {b0h, b1h, b0l, b1l} (uint4), the im half 64 B further (conflict-free
  // STS.128 / LDS.128 phases)
  auto bf_index = [&](int half, int ksub, int n, int t) {
    return half * (KSUB * K * 4 + 4) + (ksub * K + n) * 4 + (t ^ ((n >> 1) & 3));
  };
  // v (P or X: this warp's rows of its block's columns) -> B' = D^-1 v F;
  // lane pairs (g, g ^ 1) exchange so that the even lane packs the re half
  // and the odd lane the im half of rows (g & ~1, g | 1); then the pair barrier
  auto put_operand = [&](const float2 (&v)[NE], const float (&fs)[2]) {
    const bool odd = gq & 1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t hw[2], lw[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = 2 * h + c;
        const float sc2 = idsc[ie[e]] * fs[c];
        const float re = v[e].x * sc2, im = v[e].y * sc2;
        const float other = __shfl_xor_sync(0xffffffffu, odd ? re : im, 4);
        if (odd) split2(other, im, hw[h], lw[h]);  // rows (g - 1, g) of the im half
        else split2(re, other, hw[h], lw[h]);      // rows (g, g + 1) of the re half
      }
      BF[bf_index(odd ? 1 : 0, mt, je[c], gq >> 1)] = make_uint4(hw[0], hw[1], lw[0], lw[1]);
    }
    pair_sync();
  };
  // q = G v on this warp's tile (v as last put_operand'ed with column scales
  // fs): Qr = Gr Vr - Gi Vi, Qi = Gr Vi + Gi Vr
  auto product = [&](float2 (&q)[NE], const float (&ifs)[2]) {
    float acc[4][4];
#pragma unroll
    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
      for (int d = 0; d < 4; ++d) acc[a2][d] = 0.f;
    const int n = 8 * cb + gq;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint4 br = BF[bf_index(0, ks % KSUB, n, tq)], bi = BF[bf_index(1, ks % KSUB, n, tq)];
      uint4 b1 = br, b2 = bi;  // Gr block: Qr += Gr Vr, Qi += Gr Vi
      if (ks >= KSUB) {        // Gi block: Qr += Gi (-Vi), Qi += Gi Vr
        b1 = make_uint4(bi.x ^ 0x80008000u, bi.y ^ 0x80008000u, bi.z ^ 0x80008000u, bi.w ^ 0x80008000u);
        b2 = br;
      }
      hmma(acc[0], afh[ks], b1.x, b1.y);
      hmma(acc[1], afh[ks], b1.z, b1.w);
      hmma(acc[1], afl[ks], b1.x, b1.y);
      hmma(acc[2], afh[ks], b2.x, b2.y);
      hmma(acc[3], afh[ks], b2.z, b2.w);
      hmma(acc[3], afl[ks], b2.x, b2.y);
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const float u2 = idsc[ie[d]] * ifs[d & 1];  // exact: powers of two
      q[d] = make_float2((acc[0][d] + acc[1][d]) * u2, (acc[2][d] + acc[3][d]) * u2);
    }
  };

  // ---- Jac-PCG / CG (linsolve.py:217-294) on the K identity RHS, w0 = 0
  float icr[NE], icc[2], rz[2], pbm[2], pfs[2], pifs[2];
  float2 x[NE], r[NE], pv[NE], qv[NE];
  if (solver) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      icc[c] = use_c ? 1.f / cdg[je[c]] : 1.f;
      rz[c] = textbook ? icc[c] : (use_c ? icc[c] * icc[c] : 1.f);
      pbm[c] = (use_c ? icc[c] : 1.f) * idsc[je[c]];  // max_k |P0_kj| / d_k (P0 diagonal)
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
      if (direct) x[e] = gij;  // A = G + xi I, inverted in place below
    }
  }
  __syncthreads();  // G read (fragments, first product): the operand region may overwrite it
  STAMP(11);
  if (direct) {
    // ---- rzf_direct (precoder.py:73-78): X = A^-1 by in-place Gauss-Jordan
    // elimination without pivoting (A Hermitian positive definite: its pivots
    // are the squared Cholesky diagonal, so a pivot <= 0 is exactly the
    // Cholesky breakdown of linsolve.py:113-116 -> XL_STATUS_CHOLESKY).  Step
    // k publishes row k and column k (double-buffered: one barrier per step).
    float2* rowb = reinterpret_cast<float2*>(XT);  // [2][K]
    float2* colb = rowb + 2 * K;                   // [2][K]
    for (int k = 0; k < K; ++k) {
      const int buf = (k & 1) * K;
      if (solver) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          if (ie[e] == k) rowb[buf + je[e]] = x[e];
          if (je[e] == k) colb[buf + ie[e]] = x[e];
        }
      }
      __syncthreads();
      const float pk = rowb[buf + k].x;
      if (!(pk > 0.f)) {
        if (tid == 0) flags[0] |= 4;
      }
      const float ip = rcp_nr(pk);  // (a pivot <= 0 is flagged above)
      if (solver) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          // every case computed, then selected (divergent if/else chains cost
          // ~2x the step: tools/microbench/gj_step.cu)
          const int i = ie[e], j = je[e];
          const float2 a = colb[buf + i], c = rowb[buf + j];  // a_ik, a_kj (old)
          const float2 gen = make_float2(x[e].x - (a.x * c.x - a.y * c.y) * ip,
                                         x[e].y - (a.x * c.y + a.y * c.x) * ip);
          const float sr = (j == k) ? -ip : ip;  // row k: x / p, column k: -x / p
          float2 v = (i == k || j == k) ? make_float2(x[e].x * sr, x[e].y * sr) : gen;
          if (i == k && j == k) v = make_float2(ip, 0.f);
          x[e] = v;
        }
      }
    }
  } else if (solver) {
    for (int t = 1; t <= p.T; ++t) {
      if (t > 1) {
        product(qv, pifs);
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
      if (t == 1) {
        // P0 = diag(p_jj): the only non-zero term of column j's curvature is
        // p_jj (A_jj p_jj) qf_j (the sum of it and exact zeros, computed here
        // by every owner of the column without a reduction)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float pjj = use_c ? icc[c] : 1.f, qf = alg1 ? icc[c] : 1.f;
          curv[c] = pjj * ((cdg[je[c]] * pjj) * qf);
        }
      } else {
        col_sum(cp, curv, false, 0);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool act = rz[c] > 0.f;
        if (curv[c] <= 0.f && act) atomicOr(flags, 1);
        al[c] = act ? rz[c] * rcp_nr(curv[c] > 0.f ? curv[c] : 1.f) : 0.f;
      }
      float rp[NE], rm[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const float a = al[e & 1], qf = alg1 ? icr[e] : 1.f;
        x[e].x = fmaf(a, pv[e].x, x[e].x);
        x[e].y = fmaf(a, pv[e].y, x[e].y);
        r[e].x -= a * (qv[e].x * qf);
        r[e].y -= a * (qv[e].y * qf);
        const float ic = textbook ? icr[e] : 1.f;
        rp[e] = r[e].x * (r[e].x * ic) + r[e].y * (r[e].y * ic);
        rm[e] = fmaxf(fabsf(r[e].x * ic), fabsf(r[e].y * ic)) * idsc[ie[e]];
      }
      if (t == p.T) break;  // the last direction update feeds nothing
      STAMP(13 + 4 * t);
      // rz and the column max of |R C^-b| / d (one exchange: two slots, one barrier)
      float rn[2], be[2], rmx[2];
      col_red(rm[0] > rm[2] ? rm[0] : rm[2], rm[1] > rm[3] ? rm[1] : rm[3], true, 3, rmx, false);
      col_sum(rp, rn, false, 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float x0 = colx[3 * NMT * K + je[c]];
        rmx[c] = NMT > 1 ? fmaxf(x0, colx[3 * NMT * K + K + je[c]]) : rmx[c];
        be[c] = rz[c] > 0.f ? rn[c] * rcp_nr(rz[c]) : 0.f;
        rz[c] = rn[c];
        // |P_new| <= |R C^-b| + |beta| |P|, per component: the next operand's scale
        pbm[c] = rmx[c] + fabsf(be[c]) * pbm[c];
        pfs[c] = pow2s<14>(pbm[c]);
        pifs[c] = pow2_inv(pfs[c]);
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const float ic = textbook ? icr[e] : 1.f, bb = be[e & 1];
        pv[e] = make_float2(fmaf(r[e].x, ic, bb * pv[e].x), fmaf(r[e].y, ic, bb * pv[e].y));
      }
      STAMP(14 + 4 * t);
      put_operand(pv, pfs);  // the partner is past this iteration's product (barrier of slot 0)
      STAMP(15 + 4 * t);
    }
  }
  STAMP(6);

  // ---- GX = G X (own tile); ||F||^2 = Re tr(X^H GX) (fp64); SINR row partials
  float2 gx[NE];
  double sig = 0.0;
  int diag_i = -1;
  if (solver) {
    // X's exact column max (one exchange) -> its operand scale
    float xa[NE], xmx[2], xfs[2];
#pragma unroll
    for (int e = 0; e < NE; ++e) xa[e] = fmaxf(fabsf(x[e].x), fabsf(x[e].y)) * idsc[ie[e]];
    col_sum(xa, xmx, true, 4);
    float xifs[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      xfs[c] = pow2s<14>(xmx[c]);
      xifs[c] = pow2_inv(xfs[c]);
    }
    put_operand(x, xfs);  // the partner is past its last product (barrier of slot 0 in iteration T)
    product(gx, xifs);
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
      if (i == 0) tcs[j] = pow2_inv(tj);
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
  if constexpr (TC) t::fence_async_smem();
  __syncthreads();  // XT, tcs, sse
  STAMP(10);

  // ---- W = beta Z' Xe' / t_j
  if constexpr (TC) {
    // tcgen05: D_mt (TMEM cols 128 + 64 mt) = Zh Xh + Zh Xl + Zl Xh for the 128-antenna
    // tile mt; A = Z and B = Xe'^T both SWIZZLE_128B K-major (8-row groups 1024 B
    // apart, a K step of 16 components = +32 B)
    constexpr uint32_t IDW = t::idesc(128, NC, 0, 0);
    if (warp == 0) {
      t::tc_after();
      const uint32_t zh = smem_u32(Zh), zl = smem_u32(Zl), xh = smem_u32(XT), xl = xh + NC * NC * 2;
      if ((xh & 1023u) != 0) asm volatile("trap;");
      for (int mt = 0; mt < M / 128; ++mt)
#pragma unroll
        for (int ks = 0; ks < NC / 16; ++ks) {
          const uint64_t ah = sw128_desc(zh + mt * 16384 + ks * 32, 16, 1024);
          const uint64_t al = sw128_desc(zl + mt * 16384 + ks * 32, 16, 1024);
          const uint64_t bh = sw128_desc(xh + ks * 32, 16, 1024), bl = sw128_desc(xl + ks * 32, 16, 1024);
          const uint32_t d = tmem + 128 + 64 * mt;
          t::mma_w(d, ah, bh, IDW, ks > 0);
          t::mma_w(d, ah, bl, IDW, 1);
          t::mma_w(d, al, bh, IDW, 1);
        }
      t::commit_w(mbar);
    }
    t::mbar_wait(mbar, 1);
    t::tc_after();
    STAMP(7);
    // TMEM -> registers (tcgen05.ld 32x32b: thread = antenna row, 64 columns) ->
    // beta / t_j -> SWIZZLE_128B staging in the (now free) Z region: box (tile mt,
    // column half hf) = 128 rows x 128 B, 16-B chunk c of row r at c ^ (r & 7)
    // (conflict-free with a static chunk order) -> 2-D TMA tensor stores, which
    // un-swizzle into the row-major W.  (Fragment stores from registers held the
    // CTA ~3.6 k cycles at the per-SM store rate; the TMA store drains on its own.)
    const float bt = (float)btd;
    float2* Fb = p.F ? p.F + b * (int64_t)M * K : nullptr;
    for (int mt = warp >> 2; mt < M / 128; mt += 2) {
      const int r = 32 * (warp & 3) + lane, a = 128 * mt + r;
      float d[64];
      t::tmem_ld<64>(tmem + 128 + 64 * mt + ((32u * (warp & 3)) << 16), d);
      t::tmem_wait_ld();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint8_t* box = smem + (size_t)(2 * mt + hf) * 16384 + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // users 16 hf + 2 c, +1
          const int j0 = 16 * hf + 2 * c;
          const float f0 = tcs[j0], f1 = tcs[j0 + 1], w0 = bt * f0, w1 = bt * f1;
          const float* v = d + 32 * hf + 4 * c;
          *reinterpret_cast<float4*>(box + ((c ^ (r & 7)) << 4)) =
              make_float4(v[0] * w0, v[1] * w0, v[2] * w1, v[3] * w1);
          if (Fb)
            __stcs(reinterpret_cast<float4*>(Fb + (int64_t)a * K + j0),
                   make_float4(v[0] * f0, v[1] * f0, v[2] * f1, v[3] * f1));
        }
      }
    }
    t::tc_before();
    t::fence_async_smem();
    __syncthreads();  // every TMEM read done; the staged W visible to the TMA unit
    if (tid == 0) {
      const int y0 = (int)(b * M);
      for (int bx = 0; bx < 2 * (M / 128); ++bx)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&wmap)),
                     "r"(32 * (bx & 1)), "r"(y0 + 128 * (bx >> 1)), "r"(smem_u32(smem + (size_t)bx * 16384))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (warp == 0) {
      t::tc_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
  } else {
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
        const float ws = bt * its[n];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 32 * mp + 16 * h + gr;
          __stcs(Wb + (int64_t)a * K + ju, make_float2(acc[h][n][0] * ws, acc[h][n][1] * ws));
          __stcs(Wb + (int64_t)(a + 8) * K + ju, make_float2(acc[h][n][2] * ws, acc[h][n][3] * ws));
        }
      }
      if (Fb) {
#pragma unroll
        for (int n = 0; n < NTL; ++n) {
          const int ju = 4 * n + t4;
          const float it = its[n];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = 32 * mp + 16 * h + gr;
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
    if (flags[0] & 4) st = XL_STATUS_CHOLESKY;
    else if (flags[0] & 2) st = XL_STATUS_SPLITTING;
    else if (flags[0] & 1) st = XL_STATUS_NOT_HPD;
    else if (degenerate) st = XL_STATUS_DEGENERATE;
    p.status[b] = st;
    // the W tensor stores read shared memory: it must outlive them
    if constexpr (TC) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

template <int K>
size_t smem_bytes(int M) {
  using g = G<K>;
  return (size_t)M * g::NC * 2 * 2 + 2 * (size_t)K * K * 8 + g::XT_BYTES + 6 * K * 4 + (K / 8) * K * 8 +
         NW * 8 + 5 * (K / 16) * K * 4 + NW * 4 + (K + 2) * 4 + 16;
}

}  // namespace fs

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// the K = 32 variant with tcgen05 Gram / W (XL_SMALL_K_TC=0 keeps mma.sync)
bool fc64s_uses_tcgen05(int M, int K) {
  const char* tce = getenv("XL_SMALL_K_TC");
  return K == 32 && M % 128 == 0 && !(tce && tce[0] == '0');
}

bool fc64s_supported(int dtype, int method, int M, int K) {
  if (dtype != XL_C64 || (method != XL_JACPCG && method != XL_CG && method != XL_DIRECT)) return false;
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
  CUtensorMap wmap;
  memset(&wmap, 0, sizeof(wmap));
  auto launch = [&](auto kern, size_t sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fs::NT, sm);
    p.pf = (per_sm > 0 ? per_sm : 1) * nsm;
    kern<<<(unsigned)B, fs::NT, sm, st>>>(p, wmap);
  };
  // (the W tensor map addresses rows with 32-bit coordinates: beyond 2^31 rows the
  // mma.sync variant runs)
  const bool tc = fc64s_uses_tcgen05(M, K) && B * (int64_t)M <= 0x7fffffffLL;
  if (tc) {  // W [B M rows][2K floats] for the epilogue's 2-D tensor stores: boxes of 128 rows x 32 floats
    static EncodeTiled enc = nullptr;
    if (!enc) {
      void* fp = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        enc = (EncodeTiled)fp;
    }
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return XL_ERR_CUDA; }
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * K), (cuuint64_t)(B * M)};
    const cuuint64_t strides[1] = {(cuuint64_t)(2 * K) * 4};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("W tensor map encode failed");
      return XL_ERR_CUDA;
    }
  }
  if (K == 16) launch(fs::small_k_kernel<16, false>, fs::smem_bytes<16>(M));
  else if (tc) launch(fs::small_k_kernel<32, true>, fs::smem_bytes<32>(M));
  else launch(fs::small_k_kernel<32, false>, fs::smem_bytes<32>(M));
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
