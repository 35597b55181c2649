// Streaming tcgen05 Gram and W products for the large-K rzf path (complex64,
// K = 128, M % 64 == 0): the B200-native replacement of the split-operand
// library GEMMs (gemm_tc.cu tc_gram / tc_apply) for the cfg4 shape.
//
//   gram_kernel   U = Zh^T (Zh + 2 Zl) over all M antennas, Z = sz [Re H, Im H]
//                 in TMEM, emitted as A = (U + U^T)/2 + xi I (complex K x K)
//                 (sz: power of two from the first non-zero chunk; realizations
//                 whose later chunks would overflow fp16 are flagged and redone
//                 with the exact max from zmax_kernel)
//                 interleaved (M x 2K real) -- the arithmetic of
//                 gram_extract_kernel after the library GEMMs
//                 (gram_regularized, precoder.py:53-61);
//   w_kernel      W^T = beta Xe^T Z^T per realization and output half
//                 (rzf_iterative F = H X, precoder.py:90, with _power_scale's
//                 beta folded in, precoder.py:64-70), F = W / beta optional.
//
// Both streaming kernels are warp-specialised like the fused K <= 64 kernel
// (fused_tc.cu): one producer thread issues 1-D bulk copies (TMA) of 64-antenna
// raw fp32 chunks (64 KiB) into a 3-stage ring, 8 converter warps split each
// chunk in place into fp16 hi / lo core-matrix tiles (x = hi + lo, ~22
// mantissa bits), one thread issues tcgen05.mma with fp32 accumulation in
// TMEM.  Stage layout: an 8-antenna group g holds its raw rows at 8 KiB g and,
// after conversion, its hi tile at 8 KiB g and lo at 8 KiB g + 4 KiB (core
// matrix = 8 antennas x 8 components, 128 B): MN-major operands for the Gram
// (K = antennas), K-major B operand for W^T (K = components).
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>

#include "xl_common.cuh"

namespace xl {
namespace stc {

#include "tc_ptx.cuh"

constexpr int KU = 128, NC = 2 * KU;      // users, real components
constexpr int CH = 64;                    // antennas per ring stage
constexpr int SB = CH * NC * 4;           // stage bytes (64 KiB)
constexpr int NS = 3;                     // ring depth
constexpr int CMA = NC * 16;              // one fp16 tile of an 8-antenna group (4 KiB)
constexpr int GS = 2 * CMA;               // group stride (raw 8 KiB == hi + lo)
constexpr int NCONV = 8;                  // converter warps (one 8-antenna group each)
constexpr int W_PROD = 0, W_MMA = 1, W_CONV0 = 2;
constexpr int NT = 32 * (W_CONV0 + NCONV);  // 320 threads
constexpr int NIT = NC / 16;              // float4 per lane per group
constexpr int SMALL = 2048;
constexpr int SMEM = NS * SB + SMALL;
static_assert(SMEM <= 227 * 1024, "stream smem");
constexpr int BAR_CONV = 1;
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct Small {
  uint64_t raw_full[NS], conv_full[NS], stage_free[NS];
  uint64_t acc_full[2], acc_free[2];
  uint64_t done, cp_done;  // done: Gram accumulator complete / W: X columns staged
  uint32_t tmem_slot;
  float rmax[2][128];  // W: per-row partial maxima of the two k halves; Gram: converter maxima
};
static_assert(sizeof(Small) <= SMALL, "small region");

// ------------------------------------------------------------- helpers ----
// Converter lane -> (antenna row in group, component column) of iteration it:
// float4 reads and 8-B core-matrix writes bank-conflict free (fused_tc.cu).
__device__ __forceinline__ void coords(int lane, int it, int& row, int& cc) {
  const int cs = it >> 1, ih = it & 1;
  row = (lane >> 1) & 7;
  const int hb16 = lane & 1, j = (row + 2 * (lane >> 4) + ih) & 3;
  cc = 32 * cs + 8 * j + 4 * hb16;
}

// Raw fp32 group at gb -> registers (lane's share)
__device__ __forceinline__ void load_group(const uint8_t* gb, int lane, float4 (&v)[NIT]) {
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    int row, cc;
    coords(lane, it, row, cc);
    v[it] = *reinterpret_cast<const float4*>(gb + (row * NC + cc) * 4);
  }
}
// this lane's max |value| of the group (callers reduce over the warp only when needed)
__device__ __forceinline__ float lane_max(const float4 (&v)[NIT]) {
  float mx = 0.0f;
#pragma unroll
  for (int it = 0; it < NIT; ++it)
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[it].x), fabsf(v[it].y)), fmaxf(fabsf(v[it].z), fabsf(v[it].w))));
  return mx;
}
// Split the group (loaded by load_group) in place into hi / (lmul * lo) fp16 tiles.
__device__ __forceinline__ void store_group(uint8_t* gb, int lane, const float4 (&v)[NIT], float sz, float lmul) {
  __syncwarp();  // the whole group is in registers before it is overwritten
  const float2 s2 = make_float2(sz, sz), l2 = make_float2(lmul, lmul);
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    int row, cc;
    coords(lane, it, row, cc);
    const float2 a = __fmul2_rn(make_float2(v[it].x, v[it].y), s2);
    const float2 bq = __fmul2_rn(make_float2(v[it].z, v[it].w), s2);
    const __half2 ha = __float22half2_rn(a), hb = __float22half2_rn(bq);
    const float2 ra = __fadd2_rn(a, make_float2(-__low2float(ha), -__high2float(ha)));
    const float2 rb = __fadd2_rn(bq, make_float2(-__low2float(hb), -__high2float(hb)));
    const __half2 la = __float22half2_rn(__fmul2_rn(ra, l2)), lb = __float22half2_rn(__fmul2_rn(rb, l2));
    const int off = (cc >> 3) * 128 + row * 16 + (cc & 7) * 2;
    *reinterpret_cast<uint2*>(gb + off) = make_uint2(h2u(ha), h2u(hb));
    *reinterpret_cast<uint2*>(gb + CMA + off) = make_uint2(h2u(la), h2u(lb));
  }
}

// Producer (one thread): chunk c of realization b into stage c % NS.
__device__ __forceinline__ void produce(const float2* H, int64_t b, int M, uint8_t* ring, Small* sm) {
  const uint64_t pol = policy_evict_first();
  const int nch = M / CH;
  const char* src = reinterpret_cast<const char*>(H + b * (int64_t)M * KU);
  for (int c = 0; c < nch; ++c) {
    const int s = c % NS;
    if (c >= NS) mbar_wait(&sm->stage_free[s], ((c / NS) - 1) & 1);
    mbar_expect_tx(&sm->raw_full[s], SB);
    bulk_g2s(ring + s * SB, src + (int64_t)c * SB, SB, &sm->raw_full[s], pol);
  }
}

__device__ __forceinline__ void init_ring(Small* sm) {
  for (int s = 0; s < NS; ++s) {
    mbar_init(&sm->raw_full[s], 1);
    mbar_init(&sm->conv_full[s], NCONV);
    mbar_init(&sm->stage_free[s], 1);
  }
  for (int j = 0; j < 2; ++j) {
    mbar_init(&sm->acc_full[j], 1);
    mbar_init(&sm->acc_free[j], 32 * NCONV);
  }
  mbar_init(&sm->done, 1);
  mbar_init(&sm->cp_done, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ----------------------------------------------------------- zmax ---------
// grid (B), 512 threads: sz[b] = 2^e with max |sz H_b| in [2^10, 2^11), for the
// realizations flagged in only[b] (the Gram's first-chunk scale overflowed)
__global__ void __launch_bounds__(512) zmax_kernel(const float4* __restrict__ H, int64_t per4, float* __restrict__ sz,
                                                   const int* __restrict__ only) {
  const int64_t b = blockIdx.x;
  if (only && only[b] == 0) return;
  const float4* h = H + b * per4;
  float m = 0.0f;
  for (int64_t i = threadIdx.x; i < per4; i += 4 * 512) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i + u * 512 < per4) ? __ldcs(h + i + u * 512) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
  }
  __shared__ float red[16];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = red[0];
    for (int w = 1; w < 16; ++w) t = fmaxf(t, red[w]);
    sz[b] = pow2_scale(t, 11);
  }
}

// ----------------------------------------------------------- Gram ---------
// One CTA per realization.  TMEM: U rows [0, 128) at columns [0, 256), rows
// [128, 256) at [256, 512); per K-step (16 antennas) 4 MMAs of 128 x 256 x 16.
constexpr uint32_t ID_GRAM = idesc(128, NC, 1, 1);

// Scale: fixup == 0: sz from the first non-zero chunk (max |sz Z| in [2^10,
// 2^11), one more read of H saved); a later group with max |sz Z| >= 2^15
// (fp16 overflow) flags rflag[b] and the fixup launch (fixup == 1, only the
// flagged realizations, sz from zmax_kernel) recomputes U.
constexpr float RANGE_MAX = 32768.0f;

__global__ void __launch_bounds__(NT, 1) gram_kernel(const float2* __restrict__ H, int M, float* __restrict__ szv,
                                                     float2* __restrict__ A, double xi, const double* __restrict__ xi_b,
                                                     int* __restrict__ rflag, int fixup) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small* sm = reinterpret_cast<Small*>(smem + NS * SB);
  const int64_t b = blockIdx.x;
  if (fixup && rflag[b] == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = M / CH;
  if (tid == 0) init_ring(sm);
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm->tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;
  float sz = fixup ? szv[b] : 1.0f;
  if (warp == W_PROD) {
    if (lane == 0) produce(H, b, M, ring, sm);
  } else if (warp == W_MMA) {  // the whole warp issues (tcgen05 ops elect one lane)
    {
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        mbar_wait(&sm->conv_full[s], (c / NS) & 1);
        tc_after();
        const uint32_t zh = su32(ring + s * SB), zl = zh + CMA;
#pragma unroll
        for (int ks = 0; ks < CH / 16; ++ks) {
          const uint32_t o = 4 * ks * CMA;  // two groups per K-step
          const uint64_t bh = sdesc(zh + o, GS, 128), bl = sdesc(zl + o, GS, 128);
          const uint64_t a0 = bh, a1 = sdesc(zh + o + 16 * 128, GS, 128);
          mma_w(tmem, a0, bh, ID_GRAM, (c | ks) != 0);
          mma_w(tmem, a0, bl, ID_GRAM, 1);  // the lo tile holds 2 Zl
          mma_w(tmem + 256, a1, bh, ID_GRAM, (c | ks) != 0);
          mma_w(tmem + 256, a1, bl, ID_GRAM, 1);
        }
        commit_w(&sm->stage_free[s]);
      }
      commit_w(&sm->done);
    }
  } else {
    const int cw = warp - W_CONV0;
    bool have = fixup != 0, over = false;
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      mbar_wait(&sm->raw_full[s], (c / NS) & 1);
      uint8_t* gb = ring + s * SB + cw * GS;
      float4 v[NIT];
      load_group(gb, lane, v);
      float gm = lane_max(v);  // per lane: the range flag is OR-ed over the warp after the loop
      if (!have) {  // until the first non-zero chunk: max over the converter warps
        gm = warp_max(gm);
        if (lane == 0) sm->rmax[0][cw] = gm;
        named_sync(BAR_CONV, 32 * NCONV);
        float mx = sm->rmax[0][0];
#pragma unroll
        for (int w = 1; w < NCONV; ++w) mx = fmaxf(mx, sm->rmax[0][w]);
        named_sync(BAR_CONV, 32 * NCONV);
        if (mx > 0.0f) {
          sz = pow2_scale(mx, 11);
          have = true;
        }
      }
      over |= !(gm * sz < RANGE_MAX);  // also catches inf / NaN
      store_group(gb, lane, v, sz, 2.0f);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->conv_full[s]);
    }
    over = __any_sync(0xffffffffu, over);
    if (!fixup) {
      if (over && lane == 0) rflag[b] = 1;
      if (tid == 32 * W_CONV0) szv[b] = sz;
    }
    // epilogue: A = (U + U^T)/2 + xi I as complex K x K, straight from TMEM
    // (gram_regularized, precoder.py:53-61; the arithmetic of gram_extract_kernel).
    // U block (I, J) (rows 128 I.., cols 128 J..) sits at TMEM lanes 0..127,
    // columns 256 I + 128 J.  Per user-block pair (0,0), (0,1), (1,1): the
    // transposed partner block U(J, I) is staged in the (idle) ring with a padded
    // row stride, each thread (row r of block I, column half p) combines its own
    // row with the staged column, lane pairs (2i, 2i+1) form the complex entries;
    // block (1,0) is the conjugate transpose of (0,1).
    mbar_wait(&sm->done, 0);
    tc_after();
    const int q = warp & 3, p = cw >> 2;
    const int r = 32 * q + lane;
    const float isz = 1.0f / sz;  // two exact multiplies: sz^2 may overflow
    const double xi_v = xi_b ? xi_b[b] : xi;
    constexpr int SP = 129;       // staged row stride (floats): conflict-free both ways
    float* S = reinterpret_cast<float*>(ring);
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const bool odd = lane & 1;
    float2* Ab = A + b * (int64_t)KU * KU;
    const int blocks[3][2] = {{0, 0}, {0, 1}, {1, 1}};
#pragma unroll 1
    for (int bi = 0; bi < 3; ++bi) {
      const int I = blocks[bi][0], J = blocks[bi][1];
      // stage U(J, I): TMEM lane c = row c of block J, columns 256 J + 128 I ..
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        tmem_ld16(tl + 256 * J + 128 * I + 64 * p + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) S[r * SP + 64 * p + c0 + e] = v[e];
      }
      named_sync(BAR_CONV, 32 * NCONV);
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        tmem_ld16(tl + 256 * I + 128 * J + 64 * p + c0, v);  // own row r of U(I, J)
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const int c = 64 * p + c0 + e;
          const float g0 = 0.5f * (v[e] + S[c * SP + r]) * isz * isz;
          const float g1 = 0.5f * (v[e + 1] + S[(c + 1) * SP + r]) * isz * isz;
          const float p0 = __shfl_xor_sync(0xffffffffu, g0, 1), p1 = __shfl_xor_sync(0xffffffffu, g1, 1);
          float re = odd ? (p0 + g1) : (g0 + p1);
          float im = odd ? (p1 - g0) : (g1 - p0);
          const int i = 64 * I + (r >> 1), j = 64 * J + (c >> 1);
          if (i == j) {
            re = (float)((double)re + xi_v);
            im = 0.0f;
          }
          if (!odd) Ab[(int64_t)i * KU + j] = make_float2(re, im);
          else if (I != J) Ab[(int64_t)j * KU + i] = make_float2(re, -im);
        }
      }
      named_sync(BAR_CONV, 32 * NCONV);  // staged block consumed
    }
  }
  tc_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// -------------------------------------------------------------- W ---------
// CTA (b, half): output components m in [128 half, 128 half + 128).
// A operand Xe^T rows (row 2j: (Re X_ij, -Im X_ij) at k = (2i, 2i+1); row
// 2j+1: (Im X_ij, Re X_ij)), scaled per row by 2^e (max < 2^14), split and
// copied into TMEM (hi [0, 128), lo [128, 256)); accumulators (64 antennas)
// double-buffered at [256, 320) and [320, 384).
constexpr uint32_t T_AH = 0, T_AL = 128, T_ACC = 256;
constexpr uint32_t ID_W = idesc(128, CH, 0, 0);
constexpr int SBOA = NC * 16;  // K-major staging: 8-row group stride

__global__ void __launch_bounds__(NT, 1) w_kernel(const float2* __restrict__ H, int M, const float* __restrict__ szv,
                                                  const float2* __restrict__ X, const double* __restrict__ beta,
                                                  float* __restrict__ W, float* __restrict__ F) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small* sm = reinterpret_cast<Small*>(smem + NS * SB);
  const int64_t b = (int64_t)blockIdx.x >> 1;
  const int half = blockIdx.x & 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = M / CH;
  if (tid == 0) init_ring(sm);
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm->tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;
  const float sz = szv[b];
  const int q = warp & 3, cw = warp - W_CONV0, kh = cw >> 2;
  const int r = 32 * q + lane;            // local output component (TMEM lane)
  const int m = 128 * half + r;           // global output component (user column m / 2 of X)
  const bool odd = m & 1;
  float srow = 1.0f;
  // ---- stage this half's 64 columns of X (512 B of each row i) in the ring
  // above the Xe^T tiles with bulk copies, then build the split, row-scaled
  // Xe^T half from smem (converter warps)
  float2* xs = reinterpret_cast<float2*>(ring + 32 * SBOA);  // xs[i * 64 + jl]
  if (tid == 32 * W_PROD) {
    constexpr uint32_t RB = 64 * sizeof(float2);
    mbar_expect_tx(&sm->done, KU * RB);
    const float2* xsrc = X + b * (int64_t)KU * KU + 64 * half;
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < KU; ++i) bulk_g2s(xs + i * 64, xsrc + (int64_t)i * KU, RB, &sm->done, pol);
  }
  if (warp >= W_CONV0) {
    const int jl = r >> 1;  // j - 64 half
    mbar_wait(&sm->done, 0);
    float mx = 0.0f;
#pragma unroll 8
    for (int i = 64 * kh; i < 64 * kh + 64; ++i) {
      const float2 v = xs[i * 64 + jl];
      mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    sm->rmax[kh][r] = mx;
    named_sync(BAR_CONV, 32 * NCONV);
    srow = pow2_scale(fmaxf(sm->rmax[0][r], sm->rmax[1][r]), 14);
#pragma unroll 4
    for (int i0 = 64 * kh; i0 < 64 * kh + 64; i0 += 4) {  // 4 users = 8 components = one core-matrix row
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 v = xs[(i0 + u) * 64 + jl];
        split2((odd ? v.y : v.x) * srow, (odd ? v.x : -v.y) * srow, hw[u], lw[u]);
      }
      const int k = 2 * i0;
      const int o = (r >> 3) * SBOA + (k >> 3) * 128 + (r & 7) * 16;
      *reinterpret_cast<uint4*>(ring + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(ring + 16 * SBOA + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    fence_async_smem();
  }
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    const uint32_t ua = su32(ring);
#pragma unroll
    for (int s = 0; s < NC / 16; ++s) {
      tmem_cp_w(tmem + T_AH + 8 * s, sdesc(ua + 2 * s * 128, 128, SBOA));
      tmem_cp_w(tmem + T_AL + 8 * s, sdesc(ua + 16 * SBOA + 2 * s * 128, 128, SBOA));
    }
    commit_w(&sm->cp_done);
  }
  if (warp == W_PROD) {
    if (lane == 0) {
      mbar_wait(&sm->cp_done, 0);  // the staging tile (ring) has been copied
      produce(H, b, M, ring, sm);
    }
  } else if (warp == W_MMA) {  // the whole warp issues (tcgen05 ops elect one lane)
    {
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS, jb = c & 1;
        if (c >= 2) mbar_wait(&sm->acc_free[jb], ((c >> 1) - 1) & 1);
        mbar_wait(&sm->conv_full[s], (c / NS) & 1);
        tc_after();
        const uint32_t zh = su32(ring + s * SB), zl = zh + CMA;
        const uint32_t d = tmem + T_ACC + CH * jb;
#pragma unroll
        for (int ks = 0; ks < NC / 16; ++ks) {
          const uint64_t dzh = sdesc(zh + 256 * ks, 128, GS), dzl = sdesc(zl + 256 * ks, 128, GS);
          mma_ts_w(d, tmem + T_AH + 8 * ks, dzh, ID_W, ks != 0);
          mma_ts_w(d, tmem + T_AH + 8 * ks, dzl, ID_W, 1);
          mma_ts_w(d, tmem + T_AL + 8 * ks, dzh, ID_W, 1);
        }
        commit_w(&sm->stage_free[s]);
        commit_w(&sm->acc_full[jb]);
      }
    }
  } else {
    // converters: split chunk c, then drain the accumulator of chunk c - 1
    // (warps of antenna half kh: antennas 32 kh .. 32 kh + 31 of the chunk)
    const double bt = beta[b];
    const float wmul = (float)(bt / ((double)srow * (double)sz));
    const float fmul = 1.0f / (srow * sz);
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + T_ACC + 32 * kh;
    auto drain = [&](int c) {
      const int jb = c & 1;
      mbar_wait(&sm->acc_full[jb], (c >> 1) & 1);
      tc_after();
      float v[32];
      tmem_ld16(tq + CH * jb, v);
      tmem_ld16(tq + CH * jb + 16, v + 16);
      tmem_wait_ld();
      tc_before();
      mbar_arrive(&sm->acc_free[jb]);
      const int64_t n0 = (int64_t)c * CH + 32 * kh;
      float* wp = W + (b * (int64_t)M + n0) * NC + m;
#pragma unroll
      for (int n = 0; n < 32; ++n) __stcs(wp + (int64_t)n * NC, v[n] * wmul);
      if (F) {
        float* fp = F + (b * (int64_t)M + n0) * NC + m;
#pragma unroll
        for (int n = 0; n < 32; ++n) __stcs(fp + (int64_t)n * NC, v[n] * fmul);
      }
    };
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      mbar_wait(&sm->raw_full[s], (c / NS) & 1);
      uint8_t* gb = ring + s * SB + cw * GS;
      float4 v[NIT];
      load_group(gb, lane, v);
      store_group(gb, lane, v, sz, 1.0f);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->conv_full[s]);
      if (c >= 1) drain(c - 1);
    }
    drain(nch - 1);
  }
  tc_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------- W, CTA pairs ----
// w_kernel as cta_group::2 pairs (the default; XL_STREAM_W2=0 keeps w_kernel):
// the two output halves of a realization form a cluster of two and multiply
// as one M = 256 MMA (each CTA's A = its half's Xe^T rows, written into its
// own TMEM with tcgen05.st), N = 64 antennas split 32 / 32: each CTA lands and
// converts only its 32 antennas of every chunk, the pair's tensor cores read
// both halves.  Converter warps only convert (the follower's signal the
// leader's MMA issuer with CTA-scope peer arrives); a dedicated epilogue
// warpgroup drains TMEM and stores W.
namespace w2 {
constexpr int HSB = SB / 2;               // 32 KiB: this CTA's 32 antennas of a chunk
constexpr int NS2 = 6;                    // ring depth (192 KiB)
constexpr int W_EPI0 = W_CONV0 + NCONV, NEPI = 4;
constexpr int NT2 = 32 * (W_EPI0 + NEPI);  // 448 threads
constexpr int SMEM2 = NS2 * HSB + SMALL;
static_assert(SMEM2 <= 227 * 1024, "stream W2 smem");
static_assert(KU * 64 * (int)sizeof(float2) <= NS2 * HSB, "X columns staged in the ring");
constexpr uint32_t ID_W2 = idesc(256, CH, 0, 0);

struct Small2 {
  uint64_t raw_full[NS2], conv_full[NS2], stage_free[NS2];
  uint64_t acc_full[2], acc_free[2], pacc_free[2];
  uint64_t xs_done;
  uint32_t tmem_slot;
  float rmax[2][128];
};
static_assert(sizeof(Small2) <= SMALL, "stream W2 small region");

__device__ __forceinline__ void tmem_st4(uint32_t ta, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3])
               : "memory");
}

__global__ void __launch_bounds__(NT2, 1) w2_kernel(const float2* __restrict__ H, int M, const float* __restrict__ szv,
                                                    const float2* __restrict__ X, const double* __restrict__ beta,
                                                    float* __restrict__ W, float* __restrict__ F) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small2* sm = reinterpret_cast<Small2*>(smem + NS2 * HSB);
  const int64_t b = (int64_t)blockIdx.x >> 1;
  const int half = blockIdx.x & 1;  // == cluster rank
  const bool leader = half == 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = M / CH;
  if (tid == 0) {
    for (int s = 0; s < NS2; ++s) {
      mbar_init(&sm->raw_full[s], 1);
      mbar_init(&sm->conv_full[s], 2 * 4);  // leader: the 4 converter warps of the chunk in each CTA
      mbar_init(&sm->stage_free[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&sm->acc_full[j], 1);
      mbar_init(&sm->acc_free[j], NEPI);  // the local epilogue warps
      mbar_init(&sm->pacc_free[j], 1);    // leader: the follower's epilogue (relayed)
    }
    mbar_init(&sm->xs_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) tmem_alloc_pair512(&sm->tmem_slot);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;
  const float sz = szv[b];
  // ---- this half's 64 columns of X into the ring (bulk copies), then each
  // converter thread (row r, user half kh) writes its split, row-scaled Xe^T
  // entries straight into TMEM: column i of the 128 (hi) / 128 (lo) A columns
  // holds components (2i, 2i + 1) = input user i
  float2* xs = reinterpret_cast<float2*>(ring);  // xs[i * 64 + jl]
  if (tid == 32 * W_PROD) {
    constexpr uint32_t RB = 64 * sizeof(float2);
    mbar_expect_tx(&sm->xs_done, KU * RB);
    const float2* xsrc = X + b * (int64_t)KU * KU + 64 * half;
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < KU; ++i) bulk_g2s(xs + i * 64, xsrc + (int64_t)i * KU, RB, &sm->xs_done, pol);
  }
  float srow = 1.0f;
  const int q = warp & 3;
  if (warp >= W_CONV0 && warp < W_EPI0) {
    const int cw = warp - W_CONV0, kh = cw >> 2;
    const int r = 32 * q + lane;
    const int jl = r >> 1;
    const bool odd = (128 * half + r) & 1;
    mbar_wait(&sm->xs_done, 0);
    float mx = 0.0f;
#pragma unroll 8
    for (int i = 64 * kh; i < 64 * kh + 64; ++i) {
      const float2 v = xs[i * 64 + jl];
      mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    sm->rmax[kh][r] = mx;
    named_sync(BAR_CONV, 32 * NCONV);
    srow = pow2_scale(fmaxf(sm->rmax[0][r], sm->rmax[1][r]), 14);
    const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll 2
    for (int i0 = 64 * kh; i0 < 64 * kh + 64; i0 += 4) {
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 v = xs[(i0 + u) * 64 + jl];
        split2((odd ? v.y : v.x) * srow, (odd ? v.x : -v.y) * srow, hw[u], lw[u]);
      }
      tmem_st4(ta + T_AH + i0, hw);
      tmem_st4(ta + T_AL + i0, lw);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  if (warp >= W_EPI0) {  // the epilogue warps need their rows' scales too
    const int r = 32 * q + lane;
    mbar_wait(&sm->xs_done, 0);
    float mx = 0.0f;
    for (int i = 0; i < KU; ++i) {
      const float2 v = xs[i * 64 + (r >> 1)];
      mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    srow = pow2_scale(mx, 14);
  }
  tc_before();
  cluster_sync_all();  // both CTAs' A rows are in TMEM (and every barrier initialised); xs is dead
  tc_after();

  if (warp == W_PROD) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const char* src = reinterpret_cast<const char*>(H + (b * (int64_t)M + (CH / 2) * half) * KU);
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS2;
        if (c >= NS2) mbar_wait(&sm->stage_free[s], ((c / NS2) - 1) & 1);
        mbar_expect_tx(&sm->raw_full[s], HSB);
        bulk_g2s(ring + s * HSB, src + (int64_t)c * SB, HSB, &sm->raw_full[s], pol);
      }
    }
  } else if (warp == W_MMA) {
    if (leader) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS2, jb = c & 1;
        if (c >= 2) {
          mbar_wait(&sm->acc_free[jb], ((c >> 1) - 1) & 1);
          mbar_wait_cl(&sm->pacc_free[jb], ((c >> 1) - 1) & 1);
        }
        mbar_wait_cl(&sm->conv_full[s], (c / NS2) & 1);
        tc_after();
        const uint32_t zh = su32(ring + s * HSB), zl = zh + CMA;
        const uint32_t d = tmem + T_ACC + CH * jb;
#pragma unroll
        for (int ks = 0; ks < NC / 16; ++ks) {
          const uint64_t dzh = sdesc(zh + 256 * ks, 128, GS), dzl = sdesc(zl + 256 * ks, 128, GS);
          mma2_ts_w(d, tmem + T_AH + 8 * ks, dzh, ID_W2, ks != 0);
          mma2_ts_w(d, tmem + T_AH + 8 * ks, dzl, ID_W2, 1);
          mma2_ts_w(d, tmem + T_AL + 8 * ks, dzh, ID_W2, 1);
        }
        commit2_mc_w(&sm->stage_free[s], 3);
        commit2_mc_w(&sm->acc_full[jb], 3);
      }
    } else if (lane == 0) {  // relay: the follower's drain of chunk c - 2 -> the leader
      const uint32_t lead_pfree = mapa_u32(su32(&sm->pacc_free[0]), 0);
      for (int c = 2; c < nch; ++c) {
        mbar_wait(&sm->acc_free[c & 1], ((c >> 1) - 1) & 1);
        mbar_arrive_peer(lead_pfree + 8u * (uint32_t)(c & 1));
      }
    }
  } else if (warp < W_EPI0) {  // converters: 8-antenna group cw & 3 of chunks c % 2 == cw >> 2
    const int cw = warp - W_CONV0;
    const int grp = cw & 3, par = cw >> 2;
    const uint32_t conv_addr = mapa_u32(su32(&sm->conv_full[0]), 0);
    for (int c = par; c < nch; c += 2) {
      const int s = c % NS2;
      mbar_wait(&sm->raw_full[s], (c / NS2) & 1);
      uint8_t* gb = ring + s * HSB + grp * GS;
      float4 v[NIT];
      load_group(gb, lane, v);
      store_group(gb, lane, v, sz, 1.0f);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sm->conv_full[s]);
        else mbar_arrive_peer(conv_addr + 8u * (uint32_t)s);
      }
    }
  } else {  // epilogue warpgroup: lane quadrant q, the chunk's 64 antennas in two halves
    const int r = 32 * q + lane;
    const int m = 128 * half + r;
    const double bt = beta[b];
    const float wmul = (float)(bt / ((double)srow * (double)sz));
    const float fmul = 1.0f / (srow * sz);
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + T_ACC;
    for (int c = 0; c < nch; ++c) {
      const int jb = c & 1;
      mbar_wait_cl(&sm->acc_full[jb], (c >> 1) & 1);
      tc_after();
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        float v[32];
        tmem_ld16(tq + CH * jb + 32 * hh, v);
        tmem_ld16(tq + CH * jb + 32 * hh + 16, v + 16);
        tmem_wait_ld();
        if (hh == 1) {
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm->acc_free[jb]);
        }
        const int64_t n0 = (int64_t)c * CH + 32 * hh;
        float* wp = W + (b * (int64_t)M + n0) * NC + m;
#pragma unroll
        for (int n = 0; n < 32; ++n) __stcs(wp + (int64_t)n * NC, v[n] * wmul);
        if (F) {
          float* fp = F + (b * (int64_t)M + n0) * NC + m;
#pragma unroll
          for (int n = 0; n < 32; ++n) __stcs(fp + (int64_t)n * NC, v[n] * fmul);
        }
      }
    }
  }
  tc_before();
  cluster_sync_all();  // no peer arrive / multicast commit targets an exited CTA
  if (warp == W_MMA) {
    tc_after();
    tmem_free_pair512(tmem);
  }
}
}  // namespace w2

}  // namespace stc

bool stc_supported(int dtype, int M, int K) {
  if (dtype != XL_C64 || K != stc::KU || M < stc::CH || M % stc::CH != 0) return false;
  const char* e = getenv("XL_LARGE_K_GEMM");  // "library": the split-operand library GEMMs (A/B, tests)
  return !(e && e[0] == 'l');
}

// A = H^H H + xi I (B x K x K complex64) and the split scales sz[b] (rflag: B
// ints of scratch): first-chunk scales, then the fixup of the flagged realizations
int stc_gram(const void* H, int64_t B, int M, int K, double xi, const double* xi_b, float* sz, void* A, int* rflag,
             cudaStream_t st) {
  if (!stc_supported(XL_C64, M, K)) { set_error("stream Gram: unsupported shape"); return XL_ERR_UNSUPPORTED; }
  if (cudaMemsetAsync(rflag, 0, (size_t)B * sizeof(int), st) != cudaSuccess) return check_launch("stream flags");
  cudaFuncSetAttribute(stc::gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stc::SMEM);
  stc::gram_kernel<<<(unsigned)B, stc::NT, stc::SMEM, st>>>((const float2*)H, M, sz, (float2*)A, xi, xi_b, rflag, 0);
  if (int e = check_launch("stream gram")) return e;
  stc::zmax_kernel<<<(unsigned)B, 512, 0, st>>>((const float4*)H, (int64_t)M * K / 2, sz, rflag);
  if (int e = check_launch("stream zmax")) return e;
  stc::gram_kernel<<<(unsigned)B, stc::NT, stc::SMEM, st>>>((const float2*)H, M, sz, (float2*)A, xi, xi_b, rflag, 1);
  return check_launch("stream gram fixup");
}

// W = beta H X (and F = H X when F is non-null) with the scales from stc_gram
int stc_apply(const void* H, const void* X, const double* beta, const float* sz, int64_t B, int M, int K, void* W,
              void* F, cudaStream_t st) {
  if (!stc_supported(XL_C64, M, K)) { set_error("stream W: unsupported shape"); return XL_ERR_UNSUPPORTED; }
  const char* w2 = getenv("XL_STREAM_W2");  // "0": the single-CTA w_kernel (A/B, tests)
  if (!(w2 && w2[0] == '0')) {
    cudaFuncSetAttribute(stc::w2::w2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stc::w2::SMEM2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * B), 1, 1);
    cfg.blockDim = dim3(stc::w2::NT2, 1, 1);
    cfg.dynamicSmemBytes = stc::w2::SMEM2;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, stc::w2::w2_kernel, (const float2*)H, M, sz, (const float2*)X, beta, (float*)W,
                           (float*)F) != cudaSuccess)
      return check_launch("stream W2 launch");
    return check_launch("stream W2");
  }
  cudaFuncSetAttribute(stc::w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stc::SMEM);
  stc::w_kernel<<<(unsigned)(2 * B), stc::NT, stc::SMEM, st>>>((const float2*)H, M, sz, (const float2*)X, beta,
                                                               (float*)W, (float*)F);
  return check_launch("stream W");
}

}  // namespace xl
