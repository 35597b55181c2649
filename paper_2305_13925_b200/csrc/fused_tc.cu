// Fused complex64 RZF precoder on the 5th-gen tensor cores (tcgen05 + TMEM),
// warp-specialised and persistent (one CTA per SM walks over realizations).
//
// Per realization b the CTA computes, entirely on chip:
//   Gram   G = Z^T Z with Z the interleaved real embedding of H (M x 2K),
//          A = G + xi I                      (gram_regularized, precoder.py:53-61)
//   Jac-PCG / CG / Algorithm-1 with T iterations on the K identity right-hand
//          sides at once                      (linsolve.py:217-294)
//   ||F||^2 = tr(X^H G X), beta, coupling B = beta G X, SINR, sum-SE
//                                              (precoder.py:64-70, metrics.py:35-58)
//   W^T = beta Xe^T Z^T (second pass over H)  (precoder.py:90)
//
// Roles (14 warps):
//   warp 13       producer: cp.async.bulk (TMA) of raw fp32 H chunks (64
//                 antennas) into an NS-stage smem ring, for the Gram pass and
//                 again (L2-resident) for the W pass;
//   warps 0-3     converters: raw fp32 -> (hi, lo) fp16 split tiles in place;
//   warp 12       streaming MMA issuer: Gram and W tcgen05.mma per stage;
//   warps 4-11    math: A build (TMEM -> registers, warp shuffles), the PCG
//                 vector recurrences (state in registers, one RHS column per
//                 register slot), its K x K tensor-core products, beta/SINR,
//                 and the W epilogue (TMEM -> coalesced global stores).
//
// Precision ("3xFP16"): x = hi + lo, hi = fp16(x), lo = fp16(x - hi); a
// product is hi*hi' + hi*lo' + lo*hi' accumulated in fp32 in TMEM (relative
// error ~2^-22).  Operands are pre-scaled by exact powers of two (Z: first
// nonzero chunk -> max in [2^10, 2^11); A'': diag < 2^14; P, X: max < 2^14),
// which leaves every recurrence bit-equivalent to the unscaled one up to
// rounding.  A |H| dynamic range that overflows the scaling is reported as
// XL_STATUS_RANGE (the host re-runs those realizations on xl_rzf_general).
//
// smem operand layouts are the SWIZZLE_NONE canonical 8x8 fp16 core matrices
// (128 B).  One Z tile layout (core rows = antennas, 16 B rows of 8
// components) serves the Gram (MN-major A and B) and W^T (K-major B).
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "xl_common.cuh"
#include <algorithm>
#include "fused_tc.cuh"

namespace xl {
namespace tc {

#include "tc_ptx.cuh"

// ----------------------------------------------------------- geometry ----
constexpr int NCONV = 4, NMATH = 8;
constexpr int W_MMA = NCONV + NMATH, W_PROD = W_MMA + 1;
constexpr int BAR_CONV = 1, BAR_MATH = 2, BAR_EPI = 3;
// Converter warps: 0..3 plus the two spare warps of warpgroup 3 (14, 15).
#ifndef XL_GRAM2
#define XL_GRAM2 1  // Gram pass accumulates U = Zh^T (Zh + 2 Zl): 2 MMAs per K-step instead of 3
#endif
#ifndef XL_NS_MAX
#define XL_NS_MAX 3  // ring depth cap (4 stages measured 3% slower at K = 64)
#endif
// Development hooks (timing bisection bits, phase traces, L2-policy and grid
// experiments; read from XL_FUSED_* environment variables).  Off in the
// product build, where every hook folds away at compile time; tools build a
// variant with -DXL_DEV_HOOKS=1 (build_ext.py --out ... -DXL_DEV_HOOKS=1).
#ifndef XL_DEV_HOOKS
#define XL_DEV_HOOKS 0
#endif
#ifndef XL_TRACE
#define XL_TRACE XL_DEV_HOOKS  // clock64 phase stamps, enabled at run time by XL_FUSED_TRACE=<k0+1>
#endif
#ifndef XL_WB_GRAM
#define XL_WB_GRAM 1   // Gram TMEM columns double-buffer the W accumulator during W passes
#endif
#ifndef XL_WB_START
#define XL_WB_START 2  // first W chunk that may use them (A(k+1) is usually built by then)
#endif
#ifndef XL_W20
#define XL_W20 1  // K = 64: a fifth warpgroup (warps 16-19) converts and drains W^T too
#endif
// Warp layout per K.  16 warps: converters 0-3 (one 8-antenna group per chunk,
// plus the W^T epilogue) and 14, 15 (two groups).  20 warps (K = 64): eight
// converters 0-3 and 16-19, one group each, each draining half of the W^T
// accumulator of its lane quadrant; setmaxnreg moves registers from the
// streaming warpgroups (64) to the math warpgroups (136).
template <int KU>
struct Lay {
  static constexpr bool W20 = XL_W20 && KU == 64;
  static constexpr int NT = W20 ? 640 : 512;
  static constexpr int NCW = W20 ? 8 : 6;     // converter warps
  static constexpr int NEPI = W20 ? 8 : 4;    // W^T epilogue warps
  __device__ static bool is_conv(int w) { return w < NCONV || (W20 ? (w >= 16 && w < 20) : (w == 14 || w == 15)); }
  __device__ static int conv_idx(int w) { return w < NCONV ? w : (W20 ? w - 12 : w - 10); }
  __device__ static int g0(int cw) { return W20 ? cw : (cw < NCONV ? cw : NCONV + 2 * (cw - NCONV)); }
  __device__ static int ng(int cw) { return (W20 || cw < NCONV) ? 1 : 2; }
};
constexpr int NMT = 32 * NMATH;               // math threads

template <int KU>
struct Geo {
  static constexpr int NC = 2 * KU;          // real components (interleaved re/im)
#ifndef XL_CH
#define XL_CH 64
#endif
  static constexpr int CH = XL_CH;           // antennas per ring stage
  static constexpr int SB = CH * NC * 4;     // stage bytes (raw fp32 == hi + lo fp16 tiles)
  static constexpr int CMA = NC * 16;        // one fp16 tile of an 8-antenna group (hi or lo)
  // Math-written operand tiles, canonical SWIZZLE_NONE layouts, no padding:
  //  A (A'', G'', Xe; K-major, 128 rows x NC): element (n, k) at
  //    (n/8) SBOA + (k/8) 128 + (n%8) 16 + (k%8) 2 -- rows written as whole
  //    16-B core-matrix rows (uint4), conflict-free;
  //  B (P, X; MN-major, K = NC components x N = KU columns): element (k, n) at
  //    (k/8) LBOB + (n/8) 128 + (k%8) 16 + (n%8) 2 -- a thread (component k)
  //    writes 8 consecutive columns as one 16-B store, conflict-free.
  static constexpr int SBOA = NC * 16;
  static constexpr int AEPART = 16 * SBOA;        // A operand tile (128 rows)
  static constexpr int LBOB = KU * 16;
  static constexpr int PBPART = (NC / 8) * LBOB;  // B operand tile
  static constexpr int SMALL_BYTES = 3072;
  static constexpr int SLACK = NC < 128 ? 2048 : 0;  // M-padded Gram reads past the last tile
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int NS_FIT = (SMEM_MAX - 2 * AEPART - 2 * PBPART - SMALL_BYTES - SLACK) / SB;
  static constexpr int NS = NS_FIT < XL_NS_MAX ? NS_FIT : XL_NS_MAX;  // ring depth: 4 x 32 KB at K = 64
  static_assert(NS >= 3, "ring depth");
  static constexpr int OFF_AE = NS * SB + SLACK;
  static constexpr int OFF_PB = OFF_AE + 2 * AEPART;
  static constexpr int OFF_SMALL = OFF_PB + 2 * PBPART;
  static constexpr int SMEM = OFF_SMALL + SMALL_BYTES;
  static constexpr int JH = KU / 2;          // PCG columns per math thread
  static constexpr int HC = NC / 2;          // Gram columns per math thread
  static constexpr int NB = (CH / 4) * (NC / 32) / NCONV;  // converter float4 blocks per thread
  static constexpr int WH = CH / 2;          // W epilogue antennas per math thread
  static constexpr uint32_t ID_GRAM = idesc(128, NC, 1, 1);
  static constexpr uint32_t ID_W = idesc(128, CH, 0, 0);
  static constexpr uint32_t ID_P = idesc(128, KU, 0, 1);  // A'' K-major, P/X MN-major
  // TMEM columns
  // TMEM columns.  T_XE holds the A operand of the K x K products (A'' / G'')
  // and then of W^T (Xe), hi at T_XE and lo at T_XE + 64, copied in from smem
  // by tcgen05.cp so the MMAs re-read only their B operand from smem.
  static constexpr int NWB = (CH <= 32) ? 2 : 1;  // W accumulator buffers at T_W0
  static_assert(NWB * CH <= 64, "W accumulator columns");
  // XL_WB_GRAM: with one buffer at T_W0, the Gram columns (free once A(k+1)
  // is built, and until G(k+2) starts) are the second W buffer of W(k) from
  // chunk XL_WB_START on.
  static constexpr bool WB_GRAM = XL_WB_GRAM && NWB == 1;
  static constexpr uint32_t T_GRAM = 0, T_Q = 128, T_W0 = 192, T_X = 256, T_R = 320, T_XE = 384;
  static constexpr uint32_t T_W1 = NWB == 2 ? 192 + CH : T_GRAM;
  // W accumulator buffer of chunk c, the wc-th W chunk of the CTA
  __device__ static int wsel(int c, uint32_t wc) {
    if (NWB == 2) return (int)(wc & 1);
    if (!WB_GRAM) return 0;
    return (c >= XL_WB_START && ((c - XL_WB_START) & 1) == 0) ? 1 : 0;
  }
};

struct Params {
  const float2* H;
  int64_t B;
  int M;
  double xi;
  const double* xi_b;
  double power, sigma2;
  int T, method, variant;
  float2* W;
  float2* F;
  double* beta;
  double* gamma;
  double* sum_se;
  float2* X;
  int32_t* status;
  float2* dbgA;  // optional [B][K][K] regularized Gram (tests)
  int dbg;       // timing bisection bits: 1 Gram + A only, 2 no W pass, 4 no conversion,
                 // 8 no W stores, 16 no Gram MMAs (results invalid)
  long long* trace;  // optional per-phase clock64 stamps of CTA 0 (XL_FUSED_TRACE)
  int l2mode;        // L2 policy of the G-pass loads: 0 evict_first, 1 normal, 2 evict_last
  int trace_k0;      // first traced realization of CTA 0 (XL_FUSED_TRACE=k0+1)
  int stagger_ns;    // dev: odd CTAs start this much later (phase-offset experiment)
  int* counter;      // realization claim counter (workspace, zeroed per launch)
};
// the bisection bits, compile-time 0 in the product build
__device__ __forceinline__ int dbg_bits(const Params& p) { return XL_DEV_HOOKS ? p.dbg : 0; }

// Element (row n, col k) of the K-major A operand tile (core rows = n).
template <int KU>
__device__ __forceinline__ int boff(int n, int k) {
  return (n >> 3) * Geo<KU>::SBOA + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
}
// smem descriptor of K-step s (16 elements) of the A tile
template <int KU>
__device__ __forceinline__ uint64_t pdesc(uint32_t base, int s) {
  return sdesc(base + 2 * s * 128, 128, Geo<KU>::SBOA);
}
// ... and of the MN-major B tile (K-group stride LBOB, N-core stride 128)
template <int KU>
__device__ __forceinline__ uint64_t bdesc(uint32_t base, int s) {
  return sdesc(base + 2 * s * Geo<KU>::LBOB, Geo<KU>::LBOB, 128);
}

struct Small {
  uint64_t raw_full[8], conv_full[8], stage_free[8];
  uint64_t gram_full, q_full, xe_ready, scale_ready, gram_free;
  uint64_t wfull[2], wfree[2];
  uint64_t xe_consumed;  // Xe(b) copied smem -> TMEM: the smem region may hold A(b+1)
  uint64_t bq_full[4];   // realization index of pipeline slot k & 3 published
  long long bq[4];
  float wsc[2][2];       // per realization parity: W scale, F scale (for the converters' epilogue)
  uint32_t tmem_slot;
  int pad0;
  float sz_slot[2];
  float conv_red[8];
  float mred[8];
  double dred[8];
  double sse[2];        // per-warp sum-SE partials
  float cdg[64];        // Re diag of A' (no xi) per user
  float red[8 * 32];    // PCG column partials (4 quadrants x 2 halves x JH); beta step: rsq[2][128]
  float rzs[64];        // rz per column (owned by the finalising threads)
  alignas(16) float coef[2][64];  // broadcast per-column alpha / beta; beta step: dgq[128]
  alignas(16) float spx[64];  // per-column P scale 2^e (current iteration)
  alignas(16) float spy[64];  // ... and its inverse 2^-e
  __device__ float* rsq() { return red; }
  __device__ float* dgq() { return &coef[0][0]; }
};
static_assert(sizeof(Small) <= 3072, "small region");

__device__ __forceinline__ float math_max(float v, Small* sm) {
  const int mw = (threadIdx.x >> 5) - NCONV, lane = threadIdx.x & 31;
  v = warp_max(v);
  if (lane == 0) sm->mred[mw] = v;
  named_sync(BAR_MATH, NMT);
  float m = sm->mred[0];
#pragma unroll
  for (int w = 1; w < NMATH; ++w) m = fmaxf(m, sm->mred[w]);
  named_sync(BAR_MATH, NMT);
  return m;
}
__device__ __forceinline__ double math_sum_d(double v, Small* sm) {
  const int mw = (threadIdx.x >> 5) - NCONV, lane = threadIdx.x & 31;
  v = warp_sum(v);
  if (lane == 0) sm->dred[mw] = v;
  named_sync(BAR_MATH, NMT);
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NMATH; ++w) s += sm->dred[w];
  named_sync(BAR_MATH, NMT);
  return s;
}
// Column sums of per-thread partials: each warp transpose-reduces its 32
// rows, lanes < JH publish one partial per column into red[quadrant][h][j].
// The caller finalises (fixed quadrant order) after a math barrier.
template <int JH, bool MAX = false>
__device__ __forceinline__ void column_partials(float (&v)[JH], float* red, int q, int h) {
  const int lane = threadIdx.x & 31;
  float t = warp_transpose_reduce<JH, MAX>(v);
  if (lane < JH) red[(q * 2 + h) * JH + lane] = t;
}
template <int JH>
__device__ __forceinline__ float column_total(const float* red, int j) {
  const int h = j / JH, jj = j % JH;
  return ((red[(0 * 2 + h) * JH + jj] + red[(1 * 2 + h) * JH + jj]) + red[(2 * 2 + h) * JH + jj]) +
         red[(3 * 2 + h) * JH + jj];
}
template <int JH>
__device__ __forceinline__ float column_max(const float* red, int j) {
  const int h = j / JH, jj = j % JH;
  return fmaxf(fmaxf(red[(0 * 2 + h) * JH + jj], red[(1 * 2 + h) * JH + jj]),
               fmaxf(red[(2 * 2 + h) * JH + jj], red[(3 * 2 + h) * JH + jj]));
}

// 8 consecutive floats of a 32-B aligned smem array (two LDS.128)
__device__ __forceinline__ void lds8(const float* a, float (&o)[8]) {
  const float4 x = reinterpret_cast<const float4*>(a)[0], y = reinterpret_cast<const float4*>(a)[1];
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w; o[4] = y.x; o[5] = y.y; o[6] = y.z; o[7] = y.w;
}

// Write the JH columns of this thread's component row r (column j scaled by
// scl[j], or by sc1 when scl is null) as the split MN-major B operand: 8
// columns per 16-B store.
template <int KU>
__device__ __forceinline__ void write_cols(const float* v, const float* scl, float sc1, int r, int h, uint8_t* bh,
                                           uint8_t* bl) {
  constexpr int JH = Geo<KU>::JH;
#pragma unroll
  for (int g = 0; g < JH / 8; ++g) {
    float sv[8];
    if (scl) lds8(scl + h * JH + 8 * g, sv);
#pragma unroll
    for (int i = 0; i < 8; ++i) sv[i] = scl ? sv[i] : sc1;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int jj = 8 * g + 2 * i;
      split2(v[jj] * sv[2 * i], v[jj + 1] * sv[2 * i + 1], hw[i], lw[i]);
    }
    const int o = (r >> 3) * Geo<KU>::LBOB + ((h * JH) / 8 + g) * 128 + (r & 7) * 16;
    *reinterpret_cast<uint4*>(bh + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(bl + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

// Copy the K-major 128 x NC split A operand (hi, lo) from smem into TMEM
// columns [t, t + NC/2) and [t + 64, t + 64 + NC/2).  Ordered before later
// tcgen05.mma of the same thread.
// Warp-collective (all 32 lanes, one elected lane issues: see tc_ptx.cuh).
template <int KU>
__device__ __forceinline__ void cp_A(uint32_t t, uint32_t ah, uint32_t al) {
  tc_after();
#pragma unroll
  for (int s = 0; s < Geo<KU>::NC / 16; ++s) {
    tmem_cp_w(t + 8 * s, pdesc<KU>(ah, s));
    tmem_cp_w(t + 64 + 8 * s, pdesc<KU>(al, s));
  }
}

// K x K tensor-core product Q = A'' * Bop (3xFP16), both operands in smem
// (the TMEM A slot holds Xe of the previous realization while its W pass
// streams), issued by one warp (warp-collective: all 32 lanes call it).
template <int KU>
__device__ __forceinline__ void issue_kxk(uint32_t tq, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl,
                                          uint64_t* bar) {
  using G = Geo<KU>;
  tc_after();
#pragma unroll
  for (int s = 0; s < G::NC / 16; ++s) {
    const uint64_t dah = pdesc<KU>(ah, s), dal = pdesc<KU>(al, s);
    const uint64_t dbh = bdesc<KU>(bh, s), dbl = bdesc<KU>(bl, s);
    mma_w(tq, dah, dbh, G::ID_P, s != 0);
    mma_w(tq, dah, dbl, G::ID_P, 1);
    mma_w(tq, dal, dbh, G::ID_P, 1);
  }
  commit_w(bar);
}

#include "fused_math.cuh"

// ------------------------------------------------------------ kernel ----
template <int KU>
__global__ void __launch_bounds__(Lay<KU>::NT, 1) fused_rzf_kernel(Params p) {
  using G = Geo<KU>;
  constexpr int NC = G::NC, JH = G::JH, HC = G::HC, NS = G::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint8_t* aeh = smem + G::OFF_AE;
  uint8_t* ael = aeh + G::AEPART;
  uint8_t* pbh = smem + G::OFF_PB;
  uint8_t* pbl = pbh + G::PBPART;
  Small* sm = reinterpret_cast<Small*>(smem + G::OFF_SMALL);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = p.M / G::CH;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->raw_full[s], 1);
      mbar_init(&sm->conv_full[s], Lay<KU>::NCW);  // one arrival per converter warp
      mbar_init(&sm->stage_free[s], 1);
    }
    mbar_init(&sm->gram_full, 1);
    mbar_init(&sm->q_full, 1);
    mbar_init(&sm->xe_ready, 1);
    mbar_init(&sm->scale_ready, 1);
    mbar_init(&sm->gram_free, 1);
    mbar_init(&sm->xe_consumed, 1);
    for (int q = 0; q < 4; ++q) mbar_init(&sm->bq_full[q], 1);
    for (int j = 0; j < 2; ++j) {
      mbar_init(&sm->wfull[j], 1);
      mbar_init(&sm->wfree[j], 32 * Lay<KU>::NEPI);  // the W epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm->tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;
  auto cta_stamp = [&](int slot) {  // per-CTA globaltimer / clock64 (XL_FUSED_TRACE)
    if (XL_TRACE && p.trace && threadIdx.x == 0 && blockIdx.x < 256) {
      uint64_t ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      p.trace[1024 + blockIdx.x * 4 + 2 * slot] = (long long)ns;
      p.trace[1024 + blockIdx.x * 4 + 2 * slot + 1] = clock64();
    }
  };
  cta_stamp(0);

  // phase stamps (CTA 0, first 8 realizations) for pipeline analysis
  // per ring item i in [64, 128): 0 = load issued, 1 = raw landed, 2 = converted, 3 = MMAs issued
  auto item_stamp = [&](uint32_t ii, int slot) {
    const uint32_t i0 = 64 + 32 * (uint32_t)p.trace_k0;
    if (XL_TRACE && p.trace && blockIdx.x == 0 && ii >= i0 && ii < i0 + 64) p.trace[256 + (ii - i0) * 8 + slot] = clock64();
  };
  auto stamp = [&](uint32_t kk, int slot) {
    if (XL_TRACE && p.trace && blockIdx.x == 0 && kk >= (uint32_t)p.trace_k0 && kk < (uint32_t)p.trace_k0 + 8)
      p.trace[(kk - p.trace_k0) * 32 + slot] = clock64();
  };
  // 20-warp layout: 640 threads launch with 96 registers each; the streaming
  // warpgroups give theirs down to 64 so the math warpgroups can take 136
  if (Lay<KU>::W20 && (warp < NCONV || warp >= NCONV + NMATH))
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
  // Stream order of ring items (software pipeline across this CTA's
  // realizations k = 0, 1, ...):  G(0), then for every k: G(k+1), W(k).
  // G(k+1) streams while the math warps run PCG(k); W(k) needs X(k).
  // Realizations are claimed dynamically (atomic counter in the workspace):
  // the producer claims b_k just before streaming G(k) and publishes it in
  // the bq ring (4 slots: every role is within 2 realizations of the
  // producer); b_k < 0 ends the sequence.  This evens out per-SM speed
  // differences (static striding left an 11% spread of CTA end times).
  const bool is_prod = (warp == W_PROD && lane == 0);
  auto real_of = [&](uint32_t k) -> int64_t {  // b_k, or -1 past the end
    if (is_prod) {
      const int64_t b = (int64_t)atomicAdd(p.counter, 1);
      sm->bq[k & 3] = b < p.B ? b : -1;
      mbar_arrive(&sm->bq_full[k & 3]);
    } else {
      mbar_wait(&sm->bq_full[k & 3], (k >> 2) & 1);
    }
    return sm->bq[k & 3];
  };
  auto for_items = [&](auto&& body) {  // body(kk, pass, b, W pass: realization k+1 exists)
    int64_t bk = real_of(0);
    if (bk < 0) return;
    body(0u, 0, bk, false);
    for (uint32_t k = 0;; ++k) {
      const int64_t bn = real_of(k + 1);
      if (bn >= 0) body(k + 1, 0, bn, false);
      if (!(dbg_bits(p) & 3)) body(k, 1, bk, bn >= 0);
      if (bn < 0) break;
      bk = bn;
    }
  };
  if (warp == W_PROD) {
    // ------------------------------------------------------ producer ------
    if (lane == 0) {
      uint32_t i = 0;
      if (XL_DEV_HOOKS && p.stagger_ns > 0 && (blockIdx.x % 2) == 1) {
        uint64_t t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
          __nanosleep(1000);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        } while (t1 - t0 < (uint64_t)p.stagger_ns);
      }
      const uint64_t pol_first = policy_evict_first();
      const int l2m = XL_DEV_HOOKS ? p.l2mode : 0;
      const uint64_t pol_g = (l2m & 32) ? policy_keep_fraction(((l2m & 15) + 1) / 16.0f)
                             : (l2m & 3) == 0 ? pol_first
                             : (l2m & 3) == 1 ? policy_evict_normal()
                                                   : policy_evict_last();
      for_items([&](uint32_t kk, int pass, int64_t b, bool) {
        const char* Hb = reinterpret_cast<const char*>(p.H + b * (int64_t)p.M * KU);
        for (int c = 0; c < nch; ++c, ++i) {
          const int s = i % NS;
          if (i >= (uint32_t)NS) mbar_wait(&sm->stage_free[s], ((i / NS) - 1) & 1);
          item_stamp(i, 0);
          mbar_expect_tx(&sm->raw_full[s], G::SB);
          // The W pass re-reads H about two passes later; the G-pass policy
          // (l2mode) decides how hard L2 tries to keep it, the W-pass reads
          // are dead after use.
          bulk_g2s(ring + s * G::SB, Hb + (int64_t)c * G::SB, G::SB, &sm->raw_full[s],
                   pass == 0 ? pol_g : pol_first);
          if (c == 0 && pass == 0) stamp(kk, 16);
          if (c == nch - 1) stamp(kk, 17 + pass);
        }
      });
    }
  } else if (Lay<KU>::is_conv(warp)) {
    // ---------------------------------------------------- converters ------
    const int cw = Lay<KU>::conv_idx(warp);
    constexpr int NCW = Lay<KU>::NCW;
    uint32_t i = 0;
    float sz_par[2] = {1.0f, 1.0f};
    int have_par[2] = {0, 0};
    uint32_t wcv = 0;                 // W chunk counter (same sequence as the MMA issuer)
    uint32_t wuse_c[2] = {0, 0};
    const bool epi = Lay<KU>::W20 || warp < NCONV;  // the W^T epilogue warps
    auto epilogue = [&](int64_t b, int c, uint32_t kc, uint32_t item) {
      const uint32_t j = G::wsel(c, wcv);
      const uint32_t i0 = 64 + 32 * (uint32_t)p.trace_k0;
      long long* tr = (XL_TRACE && p.trace && blockIdx.x == 0 && item >= i0 && item < i0 + 64)
                          ? p.trace + 256 + (item - i0) * 8 : nullptr;
      if (Lay<KU>::W20)  // lane quadrant warp & 3; warps 0-3 the first antenna half, 16-19 the second
        w_epilogue_half<KU>(p, sm, tmem, b, c, j, wuse_c[j] & 1, kc & 1, warp >= 16 ? G::CH / 2 : 0, tr);
      else
        w_epilogue<KU>(p, sm, tmem, b, c, j, wuse_c[j] & 1, kc & 1, tr);
      ++wuse_c[j];
      ++wcv;
    };
    for_items([&](uint32_t kc, int pass, int64_t bcur, bool) {
      const int par = kc & 1;
      if (pass == 0) { sz_par[par] = 1.0f; have_par[par] = 0; }
      float sz = sz_par[par];
      int have = have_par[par];
      for (int c = 0; c < nch; ++c, ++i) {
          const int s = i % NS;
          uint8_t* st = ring + s * G::SB;
          mbar_wait(&sm->raw_full[s], (i / NS) & 1);
          if (warp == 0 && lane == 0) item_stamp(i, 1);
          // Group-interleaved stage: antenna group g (8 antennas) holds its raw
          // fp32 rows at [GS g, GS (g+1)), GS = 8 NC 4 = 2 CMA, and after
          // conversion its fp16 hi core matrices at GS g and lo at GS g + CMA,
          // i.e. the same bytes: each warp converts its own groups in place, no
          // CTA-wide barrier.  Warps 0-3 (which also run the W^T epilogue) take
          // one group, the two extra warps two.  Lane -> (row, 16-B half,
          // core matrix j) keeps the float4 reads (8-lane phases: distinct
          // (j, half)) and the uint2 writes (16-lane phases: distinct
          // (row, half)) bank-conflict free.
          constexpr int NG = G::CH / 8, GS = 2 * G::CMA, NIT = NC / 16;
          static_assert(NG == (Lay<KU>::W20 ? 8 : NCONV + 2 * 2), "group split");
          const int g0 = Lay<KU>::g0(cw), ng = Lay<KU>::ng(cw);
          auto coords = [&](int it, int& row, int& cc) {
            const int cs = it >> 1, ih = it & 1;
            row = (lane >> 1) & 7;
            const int hb16 = lane & 1, j = (row + 2 * (lane >> 4) + ih) & 3;
            cc = 32 * cs + 8 * j + 4 * hb16;
          };
          if (pass == 0 && !have) {  // until the first non-zero chunk: CTA-wide max for the scale
            float mx = 0.0f;
            for (int gi = 0; gi < ng; ++gi) {
              const uint8_t* gb = st + (g0 + gi) * GS;
#pragma unroll
              for (int it = 0; it < NIT; ++it) {
                int row, cc;
                coords(it, row, cc);
                const float4 x = *reinterpret_cast<const float4*>(gb + (row * NC + cc) * 4);
                mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
              }
            }
            mx = warp_max(mx);
            if (lane == 0) sm->conv_red[cw] = mx;
            named_sync(BAR_CONV, 32 * NCW);
            mx = sm->conv_red[0];
#pragma unroll
            for (int w = 1; w < NCW; ++w) mx = fmaxf(mx, sm->conv_red[w]);
            named_sync(BAR_CONV, 32 * NCW);
            if (mx > 0.0f) {
              sz = pow2_scale(mx, 11);  // first nonzero chunk: max |Z'| in [2^10, 2^11)
              have = 1;
            }
          }
          const float2 s2 = make_float2(sz, sz);
          for (int gi = 0; gi < ng; ++gi) {
            uint8_t* gb = st + (g0 + gi) * GS;
            float4 v[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
              int row, cc;
              coords(it, row, cc);
              v[it] = *reinterpret_cast<const float4*>(gb + (row * NC + cc) * 4);
            }
            __syncwarp();  // the whole group is in registers before it is overwritten
            if (dbg_bits(p) & 4) continue;  // dbg & 4: timing without conversion
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
              int row, cc;
              coords(it, row, cc);
              const float2 a = __fmul2_rn(make_float2(v[it].x, v[it].y), s2);
              const float2 bq = __fmul2_rn(make_float2(v[it].z, v[it].w), s2);
              const __half2 ha = __float22half2_rn(a), hb = __float22half2_rn(bq);
              const float2 ra = __fadd2_rn(a, make_float2(-__low2float(ha), -__high2float(ha)));
              const float2 rbq = __fadd2_rn(bq, make_float2(-__low2float(hb), -__high2float(hb)));
              // Gram pass with XL_GRAM2: the lo tile holds 2 Zl (exact)
              const float2 l2 = (XL_GRAM2 && pass == 0) ? make_float2(2.0f, 2.0f) : make_float2(1.0f, 1.0f);
              const __half2 la = __float22half2_rn(__fmul2_rn(ra, l2)), lb = __float22half2_rn(__fmul2_rn(rbq, l2));
              const int off = (cc >> 3) * 128 + row * 16 + (cc & 7) * 2;
              *reinterpret_cast<uint2*>(gb + off) = make_uint2(h2u(ha), h2u(hb));
              *reinterpret_cast<uint2*>(gb + G::CMA + off) = make_uint2(h2u(la), h2u(lb));
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm->conv_full[s]);  // one arrival per converter warp
          if (warp == 0 && lane == 0) {
            item_stamp(i, 2);
            if (pass == 0 && c == nch - 1) {
              sm->sz_slot[par] = sz;
              mbar_arrive(&sm->scale_ready);
            }
            if (c == 0) stamp(kc, 24 + 2 * pass);
            if (c == nch - 1) stamp(kc, 25 + 2 * pass);
          }
          // W^T epilogue of the previous chunk overlaps this chunk's MMAs
          if (pass == 1 && epi && c >= 1) {
            if (warp == 0 && lane == 0) item_stamp(i - 1, 4);
            epilogue(bcur, c - 1, kc, i - 1);
            if (warp == 0 && lane == 0) item_stamp(i - 1, 5);
          }
      }
      if (pass == 1 && epi) {
        epilogue(bcur, nch - 1, kc, i - 1);
        if (warp == 0 && lane == 0) stamp(kc, 4);
      }
      sz_par[par] = sz;
      have_par[par] = have;
    });
  } else if (warp == W_MMA) {
    // ------------------------------------------- streaming MMA issuer ------
    // the whole warp runs the loop; tcgen05 instructions elect one lane
    {
      uint32_t i = 0, wc = 0;
      uint32_t wuse[2] = {0, 0};
      for_items([&](uint32_t k, int pass, int64_t, bool has_next) {
       if (pass == 0) {
        // the TMEM Gram accumulator is free once the math warps built A(k-1)
        if (k >= 1) mbar_wait(&sm->gram_free, (k - 1) & 1);
        // ... and W epilogues that borrowed the Gram columns have drained them
        if (G::WB_GRAM && wuse[1] >= 1) mbar_wait(&sm->wfree[1], (wuse[1] - 1) & 1);
        for (int c = 0; c < nch; ++c, ++i) {  // Gram
          const int s = i % NS;
          mbar_wait(&sm->conv_full[s], (i / NS) & 1);
          if (c == 0) stamp(k, 8);
          tc_after();
          // group-interleaved stage: antenna-group (K) stride GS = 2 CMA, lo at + CMA
          const uint32_t zh = su32(ring + s * G::SB), zl = zh + G::CMA;
#pragma unroll
          for (int ks = 0; ks < G::CH / 16; ++ks) {
            if (dbg_bits(p) & 16) break;
            const uint64_t dh = sdesc(zh + 4 * ks * G::CMA, 2 * G::CMA, 128);
            const uint64_t dl = sdesc(zl + 4 * ks * G::CMA, 2 * G::CMA, 128);
            mma_w(tmem + G::T_GRAM, dh, dh, G::ID_GRAM, (c | ks) != 0);
            mma_w(tmem + G::T_GRAM, dh, dl, G::ID_GRAM, 1);            // XL_GRAM2: dl holds 2 Zl
            if (!XL_GRAM2) mma_w(tmem + G::T_GRAM, dl, dh, G::ID_GRAM, 1);
          }
          commit_w(&sm->stage_free[s]);
          item_stamp(i, 3);
        }
        commit_w(&sm->gram_full);
        stamp(k, 9);
        return;
       }
        mbar_wait(&sm->xe_ready, k & 1);
        stamp(k, 10);
        cp_A<KU>(tmem + G::T_XE, su32(aeh), su32(ael));  // Xe -> TMEM (A operand)
        commit_w(&sm->xe_consumed);  // smem Xe may now be overwritten by A(k+1)
        for (int c = 0; c < nch; ++c, ++i, ++wc) {  // W^T = Xe^T Z^T
          const int s = i % NS;
          const int j = G::wsel(c, wc);
          // first borrow of the Gram columns in W(k): A(k+1) has been built from them
          if (G::WB_GRAM && c == XL_WB_START && has_next) mbar_wait(&sm->gram_free, (k + 1) & 1);
          if (wuse[j] >= 1) mbar_wait(&sm->wfree[j], (wuse[j] - 1) & 1);
          mbar_wait(&sm->conv_full[s], (i / NS) & 1);
          tc_after();
          const uint32_t zh = su32(ring + s * G::SB), zl = zh + G::CMA;
          const uint32_t d = tmem + (j ? G::T_W1 : G::T_W0);
          const uint32_t txe = tmem + G::T_XE;
#pragma unroll
          for (int ks = 0; ks < NC / 16; ++ks) {
            const uint64_t dzh = sdesc(zh + 256 * ks, 128, 2 * G::CMA), dzl = sdesc(zl + 256 * ks, 128, 2 * G::CMA);
            mma_ts_w(d, txe + 8 * ks, dzh, G::ID_W, ks != 0);
            mma_ts_w(d, txe + 8 * ks, dzl, G::ID_W, 1);
            mma_ts_w(d, txe + 64 + 8 * ks, dzh, G::ID_W, 1);
          }
          commit_w(&sm->stage_free[s]);
          commit_w(&sm->wfull[j]);
          ++wuse[j];
          item_stamp(i, 3);
        }
        stamp(k, 11);
      });
    }
  } else if (warp < NCONV + NMATH) {
    if (Lay<KU>::W20) asm volatile("setmaxnreg.inc.sync.aligned.u32 136;");
    math_role<KU>(p, sm, aeh, ael, pbh, pbl, tmem, nch);
  }
  __syncthreads();
  cta_stamp(1);
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc

bool fused_supported(int dtype, int method, int M, int K) {
  if (dtype != XL_C64 || method == XL_DIRECT) return false;
  if (K != 16 && K != 32 && K != 64) return false;
  return M >= 64 && M % 64 == 0;
}

size_t fused_ws_bytes(int, int, int64_t, int, int) { return 256; }

static int g_num_sms = 0;

template <int KU>
static int launch_k(const tc::Params& p, cudaStream_t st) {
  constexpr int smem = tc::Geo<KU>::SMEM;
  static_assert(smem <= 227 * 1024, "fused kernel smem");
  cudaFuncSetAttribute(tc::fused_rzf_kernel<KU>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t grid = p.B < g_num_sms ? p.B : g_num_sms;
  if (XL_DEV_HOOKS)
    if (const char* e = getenv("XL_FUSED_GRID")) grid = grid < atoi(e) ? grid : atoi(e);  // scaling experiments
  tc::fused_rzf_kernel<KU><<<(unsigned)grid, tc::Lay<KU>::NT, smem, st>>>(p);
  return check_launch("fused_rzf_tc");
}

int launch_fused(int dtype, int method, int variant, const void* H, int64_t B, int M, int K,
                 double xi, const double* xi_per_batch, double power, int T, double sigma2,
                 void* W, void* F, double* beta, double* gamma, double* sum_se, void* X,
                 int32_t* status, void* ws, size_t ws_bytes, void* dbg_gram, cudaStream_t st) {
  (void)dtype;
  tc::Params p{(const float2*)H, B, M, xi, xi_per_batch, power, sigma2, T, method, variant,
               (float2*)W, (float2*)F, beta, gamma, sum_se, (float2*)X, status, (float2*)dbg_gram, 0,
               nullptr, 0};  // l2mode 0: evict_first loads, st.global.cs W stores
  p.counter = static_cast<int*>(ws);
  if (ws_bytes < sizeof(int) || cudaMemsetAsync(ws, 0, sizeof(int), st) != cudaSuccess) return check_launch("fused counter");
  if (XL_DEV_HOOKS) {
    if (const char* e = getenv("XL_FUSED_DEBUG")) p.dbg = atoi(e);
    if (const char* e = getenv("XL_FUSED_L2")) p.l2mode = atoi(e);
    if (const char* e = getenv("XL_FUSED_STAGGER")) p.stagger_ns = atoi(e);
  }
  // XL_FUSED_TRACE=1: synchronous per-phase clock64 dump of CTA 0 to stderr
  // (development aid; never set in production runs).
  static long long* trace = nullptr;
  const bool tracing = XL_TRACE && getenv("XL_FUSED_TRACE") != nullptr;
  if (tracing) p.trace_k0 = atoi(getenv("XL_FUSED_TRACE")) > 1 ? atoi(getenv("XL_FUSED_TRACE")) - 1 : 0;
  if (tracing) {
    if (!trace) cudaMalloc(&trace, 2048 * sizeof(long long));
    cudaMemsetAsync(trace, 0, 2048 * sizeof(long long), st);
    p.trace = trace;
  }
  int rc = K == 64 ? launch_k<64>(p, st) : K == 32 ? launch_k<32>(p, st) : launch_k<16>(p, st);
  if (tracing && rc == XL_SUCCESS) {
    static long long h[2048];
    cudaMemcpyAsync(h, trace, sizeof(long long) * 2048, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const long long t0 = h[16];
    static const char* names[32] = {"math:gram_full", "math:A_built", "math:pcg_done", "math:xe_ready",
                                    "math:w_epi_done", "pcg1:sp", "pcg1:mma_issue", "pcg1:q_ready",
                                    "mma:gram_start", "mma:gram_full", "mma:xe_wait_done", "mma:w_last",
                                    "pcg1:curv", "pcg1:upd", "pcg1:rz", "pcg1:P",
                                    "prod:first", "prod:G_last", "prod:W_last", "beta:sx",
                                    "beta:issue", "beta:gx", "beta:fro2", "beta:gamma",
                                    "conv:G_first", "conv:G_last", "conv:W_first", "conv:W_last",
                                    "xe:built", "xe:synced", 0, 0};
    for (int kk = 0; kk < 8; ++kk)
      for (int s = 0; s < 32; ++s)
        if (names[s] && h[kk * 32 + s]) fprintf(stderr, "trace b%d %-18s %10lld\n", kk, names[s], h[kk * 32 + s] - t0);
    {  // per-CTA wall time and effective SM clock
      long long t0n = h[1024], t1n = h[1024 + 2], mn = 1LL << 62, mx = 0;
      double clk = 0;
      int n = 0;
      for (int b = 0; b < 256 && h[1024 + 4 * b]; ++b, ++n) {
        const long long* e = h + 1024 + 4 * b;
        t0n = std::min(t0n, e[0]);
        t1n = std::max(t1n, e[2]);
        mn = std::min(mn, e[2] - e[0]);
        mx = std::max(mx, e[2] - e[0]);
        clk += (double)(e[3] - e[1]) / (double)(e[2] - e[0]);
      }
      if (n) fprintf(stderr, "ctas %d: span %.3f ms, per-CTA %.3f..%.3f ms, mean SM clock %.0f MHz\n", n, (t1n - t0n) * 1e-6,
                     mn * 1e-6, mx * 1e-6, 1e3 * clk / n);
    }
    for (int ii = 0; ii < 64; ++ii) {
      const long long* e = h + 256 + ii * 8;
      if (e[0])
        fprintf(stderr, "item %3d issue %9lld landed %9lld converted %9lld mma %9lld epi %9lld %9lld full %9lld ld %9lld\n", ii + 64,
                e[0] - t0, e[1] - t0, e[2] - t0, e[3] - t0, e[4] ? e[4] - t0 : 0, e[5] ? e[5] - t0 : 0,
                e[6] ? e[6] - t0 : 0, e[7] ? e[7] - t0 : 0);
    }
  }
  return rc;
}

}  // namespace xl
