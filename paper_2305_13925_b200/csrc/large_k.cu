// Hand-written tcgen05 chain for K = 256 (complex64, M % 64 == 0): the cfg5
// shape, where the K x K state does not fit one SM.
//
//   lk_gram_kernel  A = H^H H + xi I (gram_regularized, precoder.py:53-61).
//                   The real Gram U = Z^T Z of Z = sz [Re H, Im H] (M x 512,
//                   interleaved) in 128 x 128 tiles, upper triangle only
//                   (10 tiles), two tiles per CTA, five CTAs per realization
//                   sharing H through L2.  3xFP16: U = Zh^T Zh + Zh^T Zl +
//                   Zl^T Zh with fp32 accumulation in TMEM.  H arrives by 2-D
//                   TMA (cp.async.bulk.tensor) in 32-antenna x 128-component
//                   boxes per needed block; converter warps split each box in
//                   place into fp16 hi / lo MN-major core-matrix tiles.
//   lk_pcg_kernel   Jac-PCG / CG (linsolve.py:217-294) on a persistent
//                   8-CTA thread-block cluster per realization: CTA c owns
//                   RHS columns [32c, 32c + 32) (the K identity right-hand
//                   sides are independent columns with their own alpha_j /
//                   beta_j), keeps P in registers and Q = A''P, R and X in
//                   TMEM; the 3xFP16 split of the real embedding A''
//                   (1 MiB: does not fit one SM) is shared by the cluster --
//                   built once per realization into an L2-resident scratch
//                   slot (each CTA one eighth) and streamed to all eight
//                   CTAs' shared memory by TMA multicast (one L2 read per
//                   cluster), 32 KiB per K-step.  Also returns GX = (A - xi I)X
//                   and the ||F||^2 partials (precoder.py:64-70, metrics.py:35-44).
//   lk_w_kernel     W = beta H X (rzf_iterative F = H X, precoder.py:90):
//                   four CTAs per realization, one per 64-user output block
//                   (128 output rows, interleaved re / im).  W^T = A Zr^T +
//                   A2 Zi^T with A = [Re X; Im X]^T rows (hi, lo in TMEM) and
//                   A2 = [-Im X; Re X]^T rows (hi, lo in shared memory), Z
//                   de-interleaved into Re / Im K-steps by the converter
//                   warps; the accumulator (128 rows x 64 antennas) is
//                   double-buffered in TMEM and drained with 128-B coalesced
//                   streaming stores.
//
// Range: Z's split scale is a power of two from the first non-zero chunk
// (max |sz Z| in [2^10, 2^11)); a later group that would overflow fp16 flags
// the realization and a fixup launch redoes it with the exact maximum
// (lk_zmax_kernel), as in the K = 128 kernels (stream_tc.cu).
#include <cuda.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {
namespace lk {

#include "tc_ptx.cuh"

constexpr int KU = 256, NC = 2 * KU;
constexpr float RANGE_MAX = 32768.0f;

// ------------------------------------------------------------ PTX extras ----
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// mbarrier wait with a wall-clock bound (4 s): a protocol bug traps instead of
// hanging the GPU.  try_wait carries a suspend-time hint, so waiting warps
// sleep in hardware instead of taking issue slots from the working ones.
template <bool SPIN = false>
__device__ __forceinline__ void bwait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    if (SPIN)
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P1;\n\t}\n"
          : "=r"(done)
          : "r"(su32(bar)), "r"(parity)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, P1;\n\t}\n"
          : "=r"(done)
          : "r"(su32(bar)), "r"(parity), "r"(0x989680u)
          : "memory");
    if (done) return;
    if ((it & 15u) == 15u) {
      const uint64_t t = gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) asm volatile("trap;");
    }
  }
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 1-D bulk copy global -> the same smem offset in every CTA of `mask`,
// completing tx bytes on the mbarrier at the same offset in each
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "h"(mask)
      : "memory");
}
// arrive on the mbarrier at this offset in every CTA of `mask` when this
// thread's prior tcgen05 operations complete
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          su32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void commit_mc_w(uint64_t* bar, uint16_t mask) {  // warp-collective, one elected lane
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          su32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free512(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}
// split 8 floats (scaled) into one 16-B hi and one 16-B lo core-matrix row
__device__ __forceinline__ void split8(const float* v, float s, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split2(v[2 * i] * s, v[2 * i + 1] * s, h[i], l[i]);
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// ----------------------------------------------------------------- zmax ----
// sz[b] = 2^e with max |sz H_b| in [2^10, 2^11), for flagged realizations
__global__ void __launch_bounds__(512) lk_zmax_kernel(const float4* __restrict__ H, int64_t per4,
                                                      float* __restrict__ sz, const int* __restrict__ only) {
  const int64_t b = blockIdx.x;
  if (only[b] == 0) return;
  const float4* h = H + b * per4;
  float m = 0.0f;
  for (int64_t i = threadIdx.x; i < per4; i += 512) {
    const float4 v = __ldcs(h + i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
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

// ================================================================= Gram =====
namespace gram {
constexpr int CH = 32;                 // antennas per chunk (4 groups of 8)
constexpr int BLK = 128;               // components per block (64 users)
constexpr int SGL = CH * BLK * 4;      // 16 KiB: one block of one chunk
constexpr int PAIR = 2 * SGL;          // 32 KiB: two adjacent blocks
constexpr int SB = PAIR + SGL;         // 48 KiB per stage (at most a pair and a single)
constexpr int NS = 4;
constexpr int NCONV = 8;
constexpr int W_PROD = 0, W_MMA = 1, W_CONV0 = 2;
constexpr int NT = 32 * (W_CONV0 + NCONV);
constexpr int TPR = 5;                 // CTAs per realization
constexpr int SMALL = 1024;
constexpr int SMEM = NS * SB + SMALL;
static_assert(SMEM <= 227 * 1024, "lk gram smem");
constexpr int BAR_CONV = 1;            // 2..5: converter warp pairs of a pair group

struct Small {
  uint64_t full[NS], conv[NS], freed[NS];
  uint64_t done;
  uint32_t tmem_slot;
  float rmax[NCONV];
};
static_assert(sizeof(Small) <= SMALL, "gram small");

// CTA t of a realization: a pair slot (blocks pb, pb + 1: one 256-component
// box per chunk) and / or single slots (one 128-component box each), and its
// two 128 x 128 output tiles (I_k, J_k) at TMEM columns 128 k.  The MMA is
// N = 256 over the pair (A = its first block, or a single) where the two
// tiles share a row block, else two N = 128 products.
struct Plan {
  int pb;          // pair's first block, -1: none
  int ns, sb[2];   // singles
  int a_single;    // A operand: -1 = the pair's first block, else single index
  int I[2], J[2];
};
__constant__ Plan c_plan[TPR] = {
    {0, 0, {0, 0}, -1, {0, 0}, {0, 1}},
    {2, 1, {0, 0}, 0, {0, 0}, {2, 3}},
    {1, 0, {0, 0}, -1, {1, 1}, {1, 2}},
    {2, 0, {0, 0}, -1, {2, 2}, {2, 3}},
    {-1, 2, {1, 3}, 0, {1, 3}, {3, 3}},
};

// Conflict-free lane -> (row, component) map of a raw 8-antenna group with
// rows of 4 * NCR bytes (stc::coords): float4 reads and 8-B core-matrix
// writes hit distinct banks.
__device__ __forceinline__ void coords(int lane, int it, int& row, int& cc) {
  const int cs = it >> 1, ih = it & 1;
  row = (lane >> 1) & 7;
  const int hb16 = lane & 1, j = (row + 2 * (lane >> 4) + ih) & 3;
  cc = 32 * cs + 8 * j + 4 * hb16;
}
// load 8 float4 (iterations it0 .. it0 + 7) of a group with row stride rs bytes
__device__ __forceinline__ float load8(const uint8_t* gb, int rs, int lane, int it0, float4 (&v)[8]) {
  float mx = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int row, cc;
    coords(lane, it0 + i, row, cc);
    v[i] = *reinterpret_cast<const float4*>(gb + row * rs + cc * 4);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)), fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
  }
  return mx;
}
// split in place: hi core matrices at gb (core matrix cc >> 3 at 128 B), lo at gb + lo_off
__device__ __forceinline__ void store8(uint8_t* gb, int lo_off, int lane, int it0, const float4 (&v)[8], float sz) {
  const float2 s2 = make_float2(sz, sz);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int row, cc;
    coords(lane, it0 + i, row, cc);
    const float2 a = __fmul2_rn(make_float2(v[i].x, v[i].y), s2);
    const float2 bq = __fmul2_rn(make_float2(v[i].z, v[i].w), s2);
    const __half2 ha = __float22half2_rn(a), hb = __float22half2_rn(bq);
    const float2 ra = __fadd2_rn(a, make_float2(-__low2float(ha), -__high2float(ha)));
    const float2 rb = __fadd2_rn(bq, make_float2(-__low2float(hb), -__high2float(hb)));
    const __half2 la = __float22half2_rn(ra), lb = __float22half2_rn(rb);
    const int off = (cc >> 3) * 128 + row * 16 + (cc & 7) * 2;
    *reinterpret_cast<uint2*>(gb + off) = make_uint2(h2u(ha), h2u(hb));
    *reinterpret_cast<uint2*>(gb + lo_off + off) = make_uint2(h2u(la), h2u(lb));
  }
}

__global__ void __launch_bounds__(NT, 1) lk_gram_kernel(const __grid_constant__ CUtensorMap pmap,
                                                        const __grid_constant__ CUtensorMap smap, int M,
                                                        float* __restrict__ szv, float2* __restrict__ A, double xi,
                                                        const double* __restrict__ xi_b, int* __restrict__ rflag,
                                                        unsigned* __restrict__ zmax, int fixup) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small* sm = reinterpret_cast<Small*>(smem + NS * SB);
  const int64_t b = blockIdx.x / TPR;
  const int t = blockIdx.x % TPR;
  if (fixup && rflag[b] == 0) return;
  const Plan pl = c_plan[t];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = M / CH;
  const bool hp = pl.pb >= 0;
  const int soff = hp ? PAIR : 0;  // singles follow the pair in a stage
  const int stage_bytes = (hp ? PAIR : 0) + pl.ns * SGL;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->conv[s], NCONV);
      mbar_init(&sm->freed[s], 1);
    }
    mbar_init(&sm->done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) tmem_alloc512(&sm->tmem_slot);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sm->tmem_slot;

  if (warp == W_PROD) {
    // one lane per box of a chunk: a lane's TMA copies are serviced about one
    // at a time (tools/microbench/bulk_rules.cu), so boxes go out in parallel
    const int nbx = (hp ? 1 : 0) + pl.ns;
    if (lane < nbx) {
      const int y0 = (int)(b * M);
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        if (c >= NS) bwait<true>(&sm->freed[s], ((c / NS) - 1) & 1);
        if (lane == 0) mbar_expect_tx(&sm->full[s], stage_bytes);
        uint8_t* st = ring + s * SB;
        if (hp && lane == 0) tma2d(st, &pmap, BLK * pl.pb, y0 + c * CH, &sm->full[s]);
        else {
          const int j = lane - (hp ? 1 : 0);
          tma2d(st + soff + j * SGL, &smap, BLK * pl.sb[j], y0 + c * CH, &sm->full[s]);
        }
      }
    }
  } else if (warp == W_MMA) {  // the whole warp issues (mma_w elects one lane)
    {
      constexpr int PG = 8 * 2 * BLK * 4, SG = 8 * BLK * 4;  // group strides (8 KiB pair, 4 KiB single)
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        bwait(&sm->conv[s], (c / NS) & 1);
        tc_after();
        const uint32_t st = su32(ring + s * SB);
#pragma unroll
        for (int ks = 0; ks < CH / 16; ++ks) {
          const uint32_t acc = (c | ks) != 0;
          if (hp) {  // one N = 256 product over the pair
            const uint32_t pbase = st + 2 * ks * PG;
            uint64_t ah, al;
            if (pl.a_single < 0) {
              ah = sdesc(pbase, PG, 128);
              al = sdesc(pbase + PG / 2, PG, 128);
            } else {
              const uint32_t sbase = st + soff + pl.a_single * SGL + 2 * ks * SG;
              ah = sdesc(sbase, SG, 128);
              al = sdesc(sbase + SG / 2, SG, 128);
            }
            const uint64_t bh = sdesc(pbase, PG, 128), bl = sdesc(pbase + PG / 2, PG, 128);
            constexpr uint32_t ID256 = idesc(128, 256, 1, 1);
            mma_w(tmem, ah, bh, ID256, acc);
            mma_w(tmem, ah, bl, ID256, 1);
            mma_w(tmem, al, bh, ID256, 1);
          } else {  // two N = 128 products on singles: (A = single 0, B = single 1), (single 1, single 1)
            constexpr uint32_t ID128 = idesc(128, 128, 1, 1);
            const uint32_t s0 = st + soff + 2 * ks * SG, s1 = s0 + SGL;
            const uint64_t h0 = sdesc(s0, SG, 128), l0 = sdesc(s0 + SG / 2, SG, 128);
            const uint64_t h1 = sdesc(s1, SG, 128), l1 = sdesc(s1 + SG / 2, SG, 128);
            mma_w(tmem, h0, h1, ID128, acc);
            mma_w(tmem, h0, l1, ID128, 1);
            mma_w(tmem, l0, h1, ID128, 1);
            mma_w(tmem + 128, h1, h1, ID128, acc);
            mma_w(tmem + 128, h1, l1, ID128, 1);
            mma_w(tmem + 128, l1, h1, ID128, 1);
          }
        }
        commit_w(&sm->freed[s]);
      }
      commit_w(&sm->done);
    }
  } else {
    const int cw = warp - W_CONV0;
    float sz = fixup ? szv[b] : 1.0f;
    bool have = fixup != 0, over = false;
    float zm = 0.0f;  // exact max |H| over this CTA's blocks (the W kernel's scale)
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      bwait(&sm->full[s], (c / NS) & 1);
      uint8_t* st = ring + s * SB;
      // pair: warp cw converts half (cw & 1) of group cw >> 1 with its partner
      // warp; singles: group cw & 3 of single cw >> 2 (CTA 1: warps 0-3, single 0)
      float4 vp[8], vs[8];
      float gm = 0.0f;
      uint8_t* pg = st + (cw >> 1) * (8 * 2 * BLK * 4);
      const bool dos = hp ? (pl.ns == 1 && cw < 4) : true;
      uint8_t* sg = st + soff + (hp ? 0 : (cw >> 2) * SGL) + (cw & 3) * (8 * BLK * 4);
      if (hp) gm = load8(pg, 2 * BLK * 4, lane, 8 * (cw & 1), vp);
      if (dos) gm = fmaxf(gm, load8(sg, BLK * 4, lane, 0, vs));
      zm = fmaxf(zm, gm);  // per lane: the warp / CTA reductions happen once, after the loop
      if (!have) {  // until the first non-zero chunk: max over the converter warps
        gm = warp_max(gm);
        if (lane == 0) sm->rmax[cw] = gm;
        named_sync(BAR_CONV, 32 * NCONV);
        float mx = sm->rmax[0];
#pragma unroll
        for (int w = 1; w < NCONV; ++w) mx = fmaxf(mx, sm->rmax[w]);
        named_sync(BAR_CONV, 32 * NCONV);
        if (mx > 0.0f) {  // max in [2^6, 2^7): 2^8-2^9 x headroom for later antennas
          sz = pow2_scale(mx, 7);
          have = true;
        }
      }
      over |= !(gm * sz < RANGE_MAX);  // also catches inf / NaN
      if (hp) named_sync(2 + (cw >> 1), 64);  // both halves of the pair group are in registers
      else __syncwarp();
      if (hp) store8(pg, 8 * 2 * BLK * 2, lane, 8 * (cw & 1), vp, sz);  // lo 4 KiB after hi
      if (dos) store8(sg, 8 * BLK * 2, lane, 0, vs, sz);                 // lo 2 KiB after hi
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->conv[s]);
    }
    over = __any_sync(0xffffffffu, over);
    zm = warp_max(zm);
    if (!fixup && over && lane == 0) rflag[b] = 1;
    // the CTAs of a realization together cover every block (CTA 0: 0-1, CTA 1: 0, 2-3)
    if (lane == 0 && zm > 0.0f) atomicMax(zmax + b, __float_as_uint(zm));  // non-negative: bit order == value order
    // ---- epilogue: tile k = (I, J), lanes = rows 128 I + r, columns 128 J + c;
    // lane pairs (2i, 2i+1) form the complex entries (re = U[2i][2j] +
    // U[2i+1][2j+1], im = U[2i][2j+1] - U[2i+1][2j]); the upper triangle is
    // written with its conjugate mirror: Hermitian by construction.
    bwait(&sm->done, 0);
    tc_after();
    const int q = warp & 3, p = cw >> 2;
    const int r = 32 * q + lane;
    const float isz = 1.0f / sz;
    const double xi_v = xi_b ? xi_b[b] : xi;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const bool odd = lane & 1;
    float2* Ab = A + b * (int64_t)KU * KU;
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
      const int I = pl.I[k], J = pl.J[k];
      const int i = 64 * I + (r >> 1);
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        tmem_ld16(tl + 128 * k + 64 * p + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float g0 = v[e] * isz * isz, g1 = v[e + 1] * isz * isz;
          const float p0 = __shfl_xor_sync(0xffffffffu, g0, 1), p1 = __shfl_xor_sync(0xffffffffu, g1, 1);
          float re = odd ? (p0 + g1) : (g0 + p1);
          const float im = odd ? (p1 - g0) : (g1 - p0);
          const int j = 64 * J + ((64 * p + c0 + e) >> 1);
          if (i == j) {
            if (!odd) Ab[(int64_t)i * KU + j] = make_float2((float)((double)re + xi_v), 0.0f);
          } else if (i < j) {
            if (!odd) Ab[(int64_t)i * KU + j] = make_float2(re, im);
            else Ab[(int64_t)j * KU + i] = make_float2(re, -im);
          }
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    tmem_free512(tmem);
  }
}
}  // namespace gram

// =================================================================== W ======
namespace wk {
constexpr int CHA = 64;                  // antennas per box (MMA N)
constexpr int BU = 32;                   // users per box (64 components)
constexpr int BOX = CHA * 2 * BU * 4;    // 16 KiB
constexpr int NS = 10;                   // ring depth (160 KiB in flight)
constexpr int OFF_RING = 0;
constexpr int SBOA = KU * 16;            // K-major 8-row group stride (4 KiB)
constexpr int NCONV = 8;
constexpr int W_PROD = 0, W_MMA = 1, W_CONV0 = 2;
constexpr int NT = 32 * (W_CONV0 + NCONV);
constexpr int TPR = KU / 64;             // CTAs per realization (64 users each)
constexpr int SMALL = 2048;
constexpr int SMEM = OFF_RING + NS * BOX + SMALL;
static_assert(SMEM <= 227 * 1024, "lk W smem");
static_assert(NS * BOX >= 2 * 128 * KU * 2, "A staging fits the ring");
// TMEM: A hi / lo (the MMA A operand), then per accumulator buffer j
// D1 = A Zr^T at 256 + 128 j and D2 = A Zi^T at 256 + 128 j + 64
constexpr uint32_t T_AH = 0, T_AL = 128, T_ACC = 256;
constexpr uint32_t ID = idesc(128, CHA, 0, 0);

struct Small {
  uint64_t full[NS], conv[NS], freed[NS];
  uint64_t acc_full[2], acc_free[2];
  uint64_t cp_done;
  uint32_t tmem_slot;
  float rmax[4][64];
  float sx[64];
};
static_assert(sizeof(Small) <= SMALL, "W small");

// A-operand rows of output block t: row 2j' = Re X_{i, 64t+j'}, row 2j'+1 =
// Im X_{i, 64t+j'} over the K = 256 input users i, row j' scaled by sx[j'];
// K-major hi / lo core-matrix rows.  With D1 = A Zr^T and D2 = A Zi^T the
// output rows are W^T[2j'] = D1[2j'] - D2[2j'+1] (Re: Re X Re H - Im X Im H)
// and W^T[2j'+1] = D1[2j'+1] + D2[2j'] (Im: Im X Re H + Re X Im H).
__device__ __forceinline__ void build_rows(const float2* __restrict__ Xb, int t, const float* sx, uint8_t* dh,
                                           uint8_t* dl) {
  for (int task = threadIdx.x; task < 128 * (KU / 8); task += NT) {
    const int r = task & 127, o = task >> 7;  // row, K-octet
    const int jl = r >> 1;
    const bool odd = r & 1;
    const float s = sx[jl];
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float2 x = __ldg(Xb + (int64_t)(8 * o + e) * KU + 64 * t + jl);
      v[e] = odd ? x.y : x.x;
    }
    uint4 hi, lo;
    split8(v, s, hi, lo);
    const int off = (r >> 3) * SBOA + o * 128 + (r & 7) * 16;
    *reinterpret_cast<uint4*>(dh + off) = hi;
    *reinterpret_cast<uint4*>(dl + off) = lo;
  }
}

// zmax[b]: the exact max |H_b| (bits of a non-negative float) from lk_gram, so
// the split scale sz (max |sz H| in [2^10, 2^11)) never overflows fp16.
__global__ void __launch_bounds__(NT, 1) lk_w_kernel(const __grid_constant__ CUtensorMap hmap, int M,
                                                     const unsigned* __restrict__ zmax, const float2* __restrict__ X,
                                                     const double* __restrict__ beta, float* __restrict__ W,
                                                     float* __restrict__ F) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem + OFF_RING;
  Small* sm = reinterpret_cast<Small*>(smem + OFF_RING + NS * BOX);
  const int64_t b = blockIdx.x / TPR;
  const int t = blockIdx.x % TPR;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntile = M / CHA, nbox = ntile * (KU / BU);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->conv[s], NCONV);
      mbar_init(&sm->freed[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&sm->acc_full[j], 1);
      mbar_init(&sm->acc_free[j], 32 * NCONV);
    }
    mbar_init(&sm->cp_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) tmem_alloc512(&sm->tmem_slot);
  const float2* Xb = X + b * (int64_t)KU * KU;
  // ---- per-user scale sx[j'] = 2^e, max |X_:j'| sx < 2^14
  if (tid < 256) {
    const int jl = tid & 63, part = tid >> 6;
    float m = 0.0f;
#pragma unroll 8
    for (int i = 64 * part; i < 64 * part + 64; ++i) {
      const float2 x = __ldg(Xb + (int64_t)i * KU + 64 * t + jl);
      m = fmaxf(m, fmaxf(fabsf(x.x), fabsf(x.y)));
    }
    sm->rmax[part][jl] = m;
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (tid < 64)
    sm->sx[tid] = pow2_scale(fmaxf(fmaxf(sm->rmax[0][tid], sm->rmax[1][tid]), fmaxf(sm->rmax[2][tid], sm->rmax[3][tid])), 14);
  __syncthreads();
  const uint32_t tmem = sm->tmem_slot;
  // ---- A hi / lo staged in the (idle) ring -> TMEM
  build_rows(Xb, t, sm->sx, ring, ring + 128 * KU * 2);
  fence_async_smem();
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    const uint32_t uh = su32(ring), ul = su32(ring + 128 * KU * 2);
#pragma unroll
    for (int s = 0; s < KU / 16; ++s) {
      tmem_cp_w(tmem + T_AH + 8 * s, sdesc(uh + 2 * s * 128, 128, SBOA));
      tmem_cp_w(tmem + T_AL + 8 * s, sdesc(ul + 2 * s * 128, 128, SBOA));
    }
    commit_w(&sm->cp_done);
  }
  bwait(&sm->cp_done, 0);
  tc_after();
  __syncthreads();

  if (warp == W_PROD) {
    // lane l issues boxes g = l mod 8: a lane's TMA copies are serviced about
    // one at a time (tools/microbench/bulk_rules.cu), 8 lanes keep 8 in flight
    constexpr int NL = 8;
    if (lane < NL) {
      const int y0 = (int)(b * M);
      for (int g = lane; g < nbox; g += NL) {
        const int s = g % NS, tt = g / (KU / BU), kb = g % (KU / BU);
        if (g >= NS) bwait<true>(&sm->freed[s], ((g / NS) - 1) & 1);
        mbar_expect_tx(&sm->full[s], BOX);
        tma2d(ring + s * BOX, &hmap, 2 * BU * kb, y0 + CHA * tt, &sm->full[s]);
      }
    }
  } else if (warp == W_MMA) {  // the whole warp issues (mma_ts_w elects one lane)
    {
      for (int g = 0; g < nbox; ++g) {
        const int s = g % NS, tt = g / (KU / BU), kb = g % (KU / BU);
        if (kb == 0 && tt >= 2) bwait(&sm->acc_free[tt & 1], ((tt >> 1) - 1) & 1);
        bwait(&sm->conv[s], (g / NS) & 1);
        tc_after();
        const uint32_t st = su32(ring + s * BOX);
        const uint32_t d1 = tmem + T_ACC + 128 * (tt & 1), d2 = d1 + CHA;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int sk = 2 * kb + ks;  // K-step over input users
          const uint32_t ah = tmem + T_AH + 8 * sk, al = tmem + T_AL + 8 * sk;
          const uint64_t brh = sdesc(st + 256 * ks, 128, 2048), brl = sdesc(st + 1024 + 256 * ks, 128, 2048);
          const uint64_t bih = sdesc(st + 512 + 256 * ks, 128, 2048), bil = sdesc(st + 1536 + 256 * ks, 128, 2048);
          const uint32_t acc = (kb | ks) != 0;
          mma_ts_w(d1, ah, brh, ID, acc);
          mma_ts_w(d1, ah, brl, ID, 1);
          mma_ts_w(d1, al, brh, ID, 1);
          mma_ts_w(d2, ah, bih, ID, acc);
          mma_ts_w(d2, ah, bil, ID, 1);
          mma_ts_w(d2, al, bih, ID, 1);
        }
        commit_w(&sm->freed[s]);
        if (kb == KU / BU - 1) commit_w(&sm->acc_full[tt & 1]);
      }
    }
  } else {
    const int cw = warp - W_CONV0;
    const float sz = pow2_scale(__uint_as_float(zmax[b]), 11);
    const int crow = lane >> 2, pair = lane & 3;  // converter: antenna row of the group, user pair
    const int q = warp & 3, p = cw >> 2;
    const int r = 32 * q + lane;  // output row (TMEM lane)
    const bool odd = r & 1;
    const int col = 128 * t + r;  // output component
    const double bt = beta[b];
    const float srow = sm->sx[r >> 1];
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + T_ACC + 32 * p;
    // the scale is final from the first non-zero box on; tiles before it are all zero
    auto drain = [&](int tt) {
      const float wmul = (float)(bt / ((double)srow * (double)sz));
      const float fmul = 1.0f / (srow * sz);
      const int jb = tt & 1;
      bwait(&sm->acc_full[jb], (tt >> 1) & 1);
      tc_after();
      float v[32], u[32];
      tmem_ld16(tq + 128 * jb, v);
      tmem_ld16(tq + 128 * jb + 16, v + 16);
      tmem_ld16(tq + 128 * jb + CHA, u);
      tmem_ld16(tq + 128 * jb + CHA + 16, u + 16);
      tmem_wait_ld();
      tc_before();
      mbar_arrive(&sm->acc_free[jb]);
#pragma unroll
      for (int n = 0; n < 32; ++n) {
        const float o2 = __shfl_xor_sync(0xffffffffu, u[n], 1);
        v[n] = odd ? v[n] + o2 : v[n] - o2;
      }
      const int64_t n0 = (int64_t)tt * CHA + 32 * p;
      float* wp = W + (b * (int64_t)M + n0) * NC + col;
#pragma unroll
      for (int n = 0; n < 32; ++n) __stcs(wp + (int64_t)n * NC, v[n] * wmul);
      if (F) {
        float* fp = F + (b * (int64_t)M + n0) * NC + col;
#pragma unroll
        for (int n = 0; n < 32; ++n) __stcs(fp + (int64_t)n * NC, v[n] * fmul);
      }
    };
    for (int g = 0; g < nbox; ++g) {
      const int s = g % NS, tt = g / (KU / BU), kb = g % (KU / BU);
      bwait(&sm->full[s], (g / NS) & 1);
      uint8_t* gb = ring + s * BOX + cw * 2048;  // 8 antennas x 64 components
      // lane (row, pair) reads users 8c + 2 pair, +1 of octet c = (it + row) & 3:
      // 16-B loads and 4-B stores both bank-conflict free
      float4 v[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int c = (it + crow) & 3;
        v[it] = *reinterpret_cast<const float4*>(gb + crow * 256 + 64 * c + 16 * pair);
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int c = (it + crow) & 3;
        uint32_t hr, lr, hi_, li_;
        split2(v[it].x * sz, v[it].z * sz, hr, lr);   // Re of the user pair
        split2(v[it].y * sz, v[it].w * sz, hi_, li_); // Im
        const int o = crow * 16 + 4 * pair;
        *reinterpret_cast<uint32_t*>(gb + 128 * c + o) = hr;
        *reinterpret_cast<uint32_t*>(gb + 1024 + 128 * c + o) = lr;
        *reinterpret_cast<uint32_t*>(gb + 128 * (4 + c) + o) = hi_;
        *reinterpret_cast<uint32_t*>(gb + 1024 + 128 * (4 + c) + o) = li_;
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->conv[s]);
      if (kb == 0 && tt >= 1) drain(tt - 1);
    }
    drain(ntile - 1);
  }
  tc_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_after();
    tmem_free512(tmem);
  }
}
}  // namespace wk

// ======================================================== cluster Jac-PCG ===
namespace pc {
constexpr int C = 8;                     // CTAs per cluster
constexpr int JN = KU / C;               // RHS columns per CTA
constexpr int NT = 512;                  // 16 warps: accumulator tile w >> 2, lane quadrant w & 3
constexpr int TILE = 128 * 16 * 2;       // one 128-row x 16-K fp16 K-major operand tile (4 KiB)
constexpr int HALF = 4 * TILE;           // Re A or Im A of one K-step (2 row tiles x hi, lo): 16 KiB
constexpr int CHUNK = 2 * HALF;          // one K-step of 16 users in the scratch slot
constexpr int NCH = KU / 16;             // K-steps per product
constexpr int NB = 3 * JN;               // B tile columns: [-Pi | Pr | Pi]
constexpr int LBOB = NB * 16;            // MN-major B tile: 8-K-row group stride
constexpr int PART = (KU / 8) * LBOB;    // B tile hi or lo: 48 KiB
// Two layouts (template PR):
//  PR = false: every CTA multiplies all 256 rows of A'' by its own 32 columns
//              (M = 128 x 2 row tiles, N = 64, cta_group::1); ring stages are
//              whole K-step chunks (32 KiB), three of them.
//  PR = true:  CTA pairs (2p, 2p + 1) multiply as one cta_group::2 MMA of
//              M = 256 (CTA 2p + v supplies row tile v of A'') by N = 128 (each
//              CTA supplies its own 64 B-tile columns): each CTA lands and reads
//              only its row tile (16 KiB per K-step, five stages) and each
//              operand read feeds twice the flops.  The accumulator of CTA v
//              holds row tile v of both CTAs' columns, so the peer's half
//              (32 KiB) is exchanged through DSMEM after each product.
template <bool PR> struct Lay {
  static constexpr int STAGE = PR ? HALF : CHUNK;
  static constexpr int NS = PR ? 5 : 3;
  static constexpr int OFF_B = NS * STAGE;
  static constexpr int OFF_QX = OFF_B + 2 * PART;       // PR: the peer's Q columns, [8][256 slots][4] floats
  static constexpr int OFF_SMALL = OFF_QX + (PR ? 32768 : 0);
};
constexpr int NSMAX = 5;
// TMEM: per row tile m the accumulator [Re Q | Im Q] (2 x 32 columns) at
// 64 m; R and X in the same arrangement at 128 and 256; the A tiles of the
// current half-chunk are copied (tcgen05.cp) into one of four 32-column
// buffers at 384, so the products read A from TMEM (only B from smem)
constexpr uint32_t T_Q = 0, T_R = 128, T_X = 256, T_A = 384;
// [Re Q | Im Q] = Ar [Pr | Pi] + Ai [-Pi | Pr]: two N = 64 products per split
// part, the B operands being 64-column windows of one [-Pi | Pr | Pi] tile
constexpr uint32_t ID = idesc(128, 2 * JN, 0, 1);
constexpr uint32_t ID2 = idesc(256, 4 * JN, 0, 1);  // pair MMA: M = 256, N = 128
constexpr int BAR_MATH = 1;
constexpr size_t SLOT_BYTES = (size_t)NCH * CHUNK;  // 512 KiB of split A per cluster
// chunk layout, PR = false: [Ar: hi m0, hi m1, lo m0, lo m1 | Ai: same];
// PR = true: [row tile m0: Ar hi, Ar lo, Ai hi, Ai lo | m1: same] (a row tile is one copy)
template <bool PR>
__host__ __device__ constexpr int tile_off(int ai, int lo, int m) {
  return PR ? m * HALF + (2 * ai + lo) * TILE : ai * HALF + (2 * lo + m) * TILE;
}

struct Small {
  uint64_t full[NSMAX], empty[NSMAX], q_full;
  uint64_t pfull[NSMAX], bready, qx;  // PR: peer stage landed (leader), peer B tile ready (leader), peer Q in
  uint32_t tmem_slot;
  int not_hpd;
  float red[16][JN];
  alignas(16) float coef[2][JN];
  alignas(16) float spx[JN];
  alignas(16) float spy[JN];
  float rzs[JN];
  float cdg[KU];
  float dmax[16];
  double dred[16];
};
template <bool PR> constexpr int smem_bytes() { return Lay<PR>::OFF_SMALL + (int)sizeof(Small); }
template <bool PR> constexpr int cl_size() { return PR ? 4 : C; }  // CTAs per cluster
constexpr int MAX_SLOTS = 64;  // scratch slots (one per resident cluster)
static_assert(smem_bytes<false>() <= 227 * 1024 && smem_bytes<true>() <= 227 * 1024, "lk pcg smem");
static_assert(Lay<false>::NS * Lay<false>::STAGE >= KU * (2 * JN + 1) * 4 &&
                  Lay<true>::NS * Lay<true>::STAGE >= KU * (2 * JN + 1) * 4,
              "X / GX staging fits the ring");
static_assert(Lay<true>::NS <= NSMAX && Lay<false>::NS <= NSMAX, "ring barriers");

// ---- cta_group::2 forms: tc_ptx.cuh (mma2_w, commit2_mc_w, mapa_u32, mbar_arrive_peer, ...)
template <bool PR>
__device__ __forceinline__ void tmem_alloc512_g(uint32_t* slot) {
  if (PR) {
    tmem_alloc_pair512(slot);
  } else {
    tmem_alloc512(slot);
  }
}
template <bool PR>
__device__ __forceinline__ void tmem_free512_g(uint32_t t) {
  if (PR) tmem_free_pair512(t);
  else tmem_free512(t);
}
// wait with acquire at cluster scope (the phase was completed from another CTA)
__device__ __forceinline__ void bwait_cl(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
    if (done) return;
    if ((it & 15u) == 15u) {
      const uint64_t t = gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) asm volatile("trap;");
    }
  }
}
__device__ __forceinline__ void st_async_v4(uint32_t cl_addr, const float* v, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cl_addr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(cl_bar)
               : "memory");
}

struct Params {
  const float2* A;  // [B][K][K] regularized Gram (Hermitian, xi on the diagonal)
  int64_t B;
  int T, method, variant;
  double xi;
  const double* xi_b;
  float2* X;        // [B][K][K]
  float2* GX;       // [B][K][K]
  double* part;     // [B][C] Re tr(X^H GX) per CTA
  double* rsq;      // [B][C][2][K] per (column block, part) row sums of GX^2, or null: GX written instead
  float2* gdiag;    // [B][K] diagonal of GX (with rsq)
  float* xmax;      // [B][K] max_i max(|Re X_ij|, |Im X_ij|) per column j (the W kernel's scales), or null
  int32_t* status;  // [B]
  uint8_t* scratch; // [clusters][512 KiB] split (Re A, Im A), K-step chunks
  long long* trace; // debug: clock64 stamps of cluster 0 / CTA 0 (xl_debug_lk_trace), or null
  int unicast;      // 1: every CTA loads every chunk itself (no multicast; A/B)
  int mma_reps;     // debug: issue each K-step's MMAs this many times (timing experiments)
  int ss;           // 1: A operand straight from shared memory (no tcgen05.cp to TMEM)
  int spin;         // 1: the MMA warp polls the ring barriers without a suspend hint
};

__device__ __forceinline__ void lds8(const float* a, float (&o)[8]) {
  const float4 x = reinterpret_cast<const float4*>(a)[0], y = reinterpret_cast<const float4*>(a)[1];
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w; o[4] = y.x; o[5] = y.y; o[6] = y.z; o[7] = y.w;
}
// per-thread column values -> red[warp][lane] (warp transpose-reduce)
template <bool MAX = false>
__device__ __forceinline__ void col_partials(float (&v)[JN], Small* sm, int warp) {
  const float t = warp_transpose_reduce<JN, MAX>(v);
  sm->red[warp][threadIdx.x & 31] = t;
}
// CTA total of column j over the 16 warps in a fixed order
template <bool MAX = false>
__device__ __forceinline__ float col_total(const Small* sm, int j) {
  float s = sm->red[0][j];
#pragma unroll
  for (int w = 1; w < 16; ++w) s = MAX ? fmaxf(s, sm->red[w][j]) : s + sm->red[w][j];
  return s;
}

// One cluster of 8 CTAs per realization (persistent over b); CTA c owns RHS
// columns [32c, 32c + 32).  Thread (tile tau = warp >> 2, quadrant q, lane)
// owns component (user u = 128 (tau & 1) + 32 q + lane, part = tau >> 1:
// 0 = Re, 1 = Im) of its 32 columns: P in registers, Q / R / X in TMEM.
// Q = A P as complex products of the streamed split Re A / Im A tiles:
// Re Q = Ar Pr - Ai Pi, Im Q = Ar Pi + Ai Pr (3xFP16 each: 24 MMAs per K-step).
template <bool PR>
__global__ void __launch_bounds__(NT, 1) lk_pcg_kernel(Params p) {
  using L = Lay<PR>;
  constexpr int NS = L::NS;
  // PR: clusters of CL = 4 CTAs (two pairs) each take one half of a
  // realization's 256 RHS columns (work item = (b, half)), so 4-CTA clusters
  // tile more of the 148 SMs than 8-CTA ones; each builds the whole split A''.
  constexpr int CL = PR ? 4 : C;
  constexpr int UPC = KU / CL;  // users of the split A'' this CTA builds
  constexpr uint16_t ALL = (uint16_t)((1u << CL) - 1u);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint8_t* pb = smem + L::OFF_B;
  float* qxb = reinterpret_cast<float*>(smem + L::OFF_QX);
  Small* sm = reinterpret_cast<Small*>(smem + L::OFF_SMALL);
  const uint32_t rank = cluster_rank();
  const uint32_t cid = cluster_id_x(), ncl = nclusters_x();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tau = warp >> 2, q = warp & 3;
  const int u = 128 * (tau & 1) + 32 * q + lane;  // user of the thread's component
  const int part = tau >> 1;                      // 0: Re, 1: Im
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  uint8_t* slot = p.scratch + (size_t)cid * SLOT_BYTES;
  // PR: pair rank v (row tile of A'' this CTA supplies / its accumulator holds);
  // a thread whose user u lies in the other row tile gets its Q from the peer
  const uint32_t pr = rank & 1u, peer = rank ^ 1u;
  const bool leader = pr == 0;
  const bool remote = PR && (uint32_t)(tau & 1) != pr;
  const int qslot = part * 128 + q * 32 + lane;  // PR: exchange slot (same in sender and receiver)
  const uint16_t pair_mask = (uint16_t)(3u << (rank & ~1u));
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->empty[s], PR ? (p.unicast ? 1 : CL / 2) : (p.unicast ? 1 : C));
      mbar_init(&sm->pfull[s], 1);
    }
    mbar_init(&sm->q_full, 1);
    mbar_init(&sm->bready, 1);
    mbar_init(&sm->qx, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc512_g<PR>(&sm->tmem_slot);
  tc_before();
  __syncthreads();
  tc_after();
  if (PR) cluster_sync();  // every CTA's barriers are initialised before any remote arrive / multicast
  const uint32_t tmem = sm->tmem_slot;
  const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
  // PR: the accumulator columns of pair CTA w's B half are [64 w, 64 w + 64), so
  // the same offset reads this thread's own Q (local) or the peer's (to send)
  const uint32_t tcol = 2 * JN * (tau & 1) + JN * (tau >> 1);
  const uint32_t tQ = tl + T_Q + tcol, tR = tl + T_R + tcol, tX = tl + T_X + tcol;
  const uint32_t upb = su32(pb);
  const uint32_t peer_qx = PR ? mapa_u32(su32(qxb), peer) : 0u;
  const uint32_t peer_qxbar = PR ? mapa_u32(su32(&sm->qx), peer) : 0u;
  const uint32_t lead_pfull = PR ? mapa_u32(su32(&sm->pfull[0]), rank & ~1u) : 0u;
  const uint32_t lead_bready = PR ? mapa_u32(su32(&sm->bready), rank & ~1u) : 0u;
  uint32_t g_prod = 0, g_cons = 0, nq = 0;  // ring chunks produced / consumed, products
  // the producer warp streams the split A: chunk n of the item's (T - 1) x 16
  // K-steps into ring stage g % NS of every CTA of the cluster, armed in every
  // CTA, copied by its owner with one multicast once every consumer has freed
  // the stage (PR: each pair rank gets its own 16 KiB row tile, owner CTA
  // 2 (k % (CL / 2)) + rank parity; else the whole 32 KiB chunk, owner k % 8)
  int n_issued = 0, n_total = 0;
  // (called by all lanes of warp 1; lane 0 does the barrier / copy work)
  // a lane's bulk copies are serviced about one at a time, so the fill rate
  // grows with the copy size (tools/microbench/bulk_rules.cu)
  auto issue_next = [&]() {  // chunk n: K-step n % NCH
    if (n_issued >= n_total) return;
    const int s = g_prod % NS, k = n_issued % NCH;
    const uint8_t* src = slot + (size_t)k * CHUNK;
    if (lane == 0) {
      if (g_prod >= NS) bwait<true>(&sm->empty[s], ((g_prod / NS) - 1) & 1);
      if (p.trace && cid == 0 && rank == 0 && g_prod < 64) p.trace[128 + g_prod] = clock64();
      mbar_expect_tx(&sm->full[s], L::STAGE);
      if (PR) {  // row tile pr of K-step k, to the CTAs of this pair rank, by CTA 2 (k % (CL / 2)) + pr
        if (p.unicast)  // every CTA loads its own row tile; stages freed by its pair's MMAs only
          bulk_g2s(ring + s * L::STAGE, src + pr * HALF, HALF, &sm->full[s], policy_evict_normal());
        else if ((k % (CL / 2)) == (int)(rank >> 1))
          bulk_mc(ring + s * L::STAGE, src + pr * HALF, HALF, &sm->full[s], (uint16_t)((pr ? 0xAAAA : 0x5555) & ALL));
      } else if (p.unicast) {
        bulk_g2s(ring + s * CHUNK, src, CHUNK, &sm->full[s], policy_evict_normal());
      } else if ((k & (C - 1)) == (int)rank) {
        bulk_mc(ring + s * CHUNK, src, CHUNK, &sm->full[s], 0xFF);
      }
    }
    __syncwarp();
    ++g_prod;
    ++n_issued;
  };

  const bool tr = p.trace && cid == 0 && rank == 0 && tid == 0;
  int ntr = 0;
  auto stamp = [&]() {
    if (tr && ntr < 128) p.trace[ntr++] = clock64();
  };
  const int64_t nitems = PR ? 2 * p.B : p.B;
  for (int64_t item = cid; item < nitems; item += ncl) {
    const int64_t b = PR ? item >> 1 : item;
    const int cb = PR ? 4 * (int)(item & 1) + (int)rank : (int)rank;  // the CTA's 32-column block
    const float2* a = p.A + b * (int64_t)KU * KU;
    stamp();
    cluster_sync();  // the previous realization's chunks are consumed in every CTA
    stamp();
    // ---- scale: diag(A) sa < 2^14; zero diagonal -> Splitting (linsolve.py:205-208)
    if (tid < KU) sm->cdg[tid] = a[(int64_t)tid * KU + tid].x;
    if (tid == 0) sm->not_hpd = 0;
    __syncthreads();
    if (warp < KU / 32) {
      const float d = sm->cdg[tid];
      const float mx = warp_max(fabsf(d));
      const unsigned z = __ballot_sync(0xffffffffu, use_c && d == 0.0f);
      if (lane == 0) {
        sm->dmax[warp] = mx;
        sm->dmax[8 + warp] = z ? 1.0f : 0.0f;
      }
    }
    __syncthreads();
    float dmax = sm->dmax[0], zsum = sm->dmax[8];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      dmax = fmaxf(dmax, sm->dmax[w]);
      zsum += sm->dmax[8 + w];
    }
    const float sa = pow2_scale(dmax, 14);
    // ---- this CTA's K-step chunks (users k in [UPC rank, UPC rank + UPC)) of
    // the split (Re A, Im A) -> the cluster's scratch slot, K-major core
    // matrices; a_ik = conj(A[k][i]) (A Hermitian): Re = A[k][i].x, Im = -A[k][i].y
    for (int task = tid; task < KU * (UPC / 8); task += NT) {
      const int i = task & (KU - 1), ko = task >> 8;  // row, K-octet of the CTA's UPC users
      float vr[8], vi[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float2 x = __ldg(a + (int64_t)(UPC * (int)rank + 8 * ko + e) * KU + i);
        vr[e] = x.x;
        vi[e] = -x.y;
      }
      uint4 hr, lr, hi_, li_;
      split8(vr, sa, hr, lr);
      split8(vi, sa, hi_, li_);
      const int s = (UPC / 16) * (int)rank + (ko >> 1), kg = ko & 1, m = i >> 7;
      uint8_t* dst = slot + (size_t)s * CHUNK + ((i & 127) >> 3) * 256 + kg * 128 + (i & 7) * 16;
      *reinterpret_cast<uint4*>(dst + tile_off<PR>(0, 0, m)) = hr;
      *reinterpret_cast<uint4*>(dst + tile_off<PR>(0, 1, m)) = lr;
      *reinterpret_cast<uint4*>(dst + tile_off<PR>(1, 0, m)) = hi_;
      *reinterpret_cast<uint4*>(dst + tile_off<PR>(1, 1, m)) = li_;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    stamp();
    cluster_sync();  // the whole split A is in the slot
    stamp();
    if (warp == 1) {  // the producer warp of the product phases
      n_issued = 0;
      n_total = (p.T - 1) * NCH;  // T - 1 products (the first is a column scaling, GX comes from the residual)
      for (int i = 0; i < NS; ++i) issue_next();
    }

    const float cr = use_c ? sm->cdg[u] * sa : 1.0f;
    const float icr = 1.0f / cr;
    const double alpha = p.xi_b ? p.xi_b[b] : p.xi;
    // ---- initial state (linsolve.py:224-229, 264-268): x = 0, r = I (Algorithm 1:
    // C^-1 I), m = z, rz per column
    float P[JN], A[JN];
#pragma unroll
    for (int c0 = 0; c0 < JN; c0 += 8) {
      float rv[8], zx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int jg = JN * cb + c0 + i;
        const float e = (part == 0 && u == jg) ? 1.0f : 0.0f;
        rv[i] = (use_c && !textbook) ? e * icr : e;
        P[c0 + i] = textbook ? e * icr : rv[i];
        zx[i] = 0.0f;
      }
      tmem_st8(tR + c0, rv);
      tmem_st8(tX + c0, zx);
    }
    if (tid < JN) {
      const float c0 = use_c ? sm->cdg[JN * cb + tid] * sa : 1.0f;
      const float ic = 1.0f / c0;
      sm->rzs[tid] = textbook ? ic : (use_c ? ic * ic : 1.0f);
    }
    tmem_wait_st();

    // column max over the CTA -> spx / spy (power-of-two scale of the fp16 split, < 2^14)
    auto scale = [&](float (&v)[JN]) {
#pragma unroll
      for (int jj = 0; jj < JN; ++jj) A[jj] = fabsf(v[jj]);
      col_partials<true>(A, sm, warp);
      named_sync(BAR_MATH, NT);
      if (tid < JN) {
        const float s = pow2_scale(col_total<true>(sm, tid), 14);
        sm->spx[tid] = s;
        sm->spy[tid] = 1.0f / s;
      }
      named_sync(BAR_MATH, NT);
    };
    // Q = A v (v scaled per column): B tiles (Pr, Pi; hi, lo) written by all,
    // MMAs issued by thread 0
    auto product = [&](const float (&v)[JN]) {
      if (PR && tid == 0) mbar_expect_tx(&sm->qx, 32768);  // this product's peer Q (before our B-ready)
      // B tile columns [-Pi | Pr | Pi]: Re rows write Pr, Im rows write Pi and -Pi
#pragma unroll
      for (int g = 0; g < JN / 8; ++g) {
        float sv[8], w8[8];
        lds8(sm->spx + 8 * g, sv);
#pragma unroll
        for (int i = 0; i < 8; ++i) w8[i] = v[8 * g + i] * sv[i];
        uint4 hi, lo;
        split8(w8, 1.0f, hi, lo);
        const int o = (u >> 3) * LBOB + (u & 7) * 16;
        if (part == 0) {
          *reinterpret_cast<uint4*>(pb + o + (4 + g) * 128) = hi;
          *reinterpret_cast<uint4*>(pb + PART + o + (4 + g) * 128) = lo;
        } else {
          const uint4 nh = make_uint4(hi.x ^ 0x80008000u, hi.y ^ 0x80008000u, hi.z ^ 0x80008000u, hi.w ^ 0x80008000u);
          const uint4 nl = make_uint4(lo.x ^ 0x80008000u, lo.y ^ 0x80008000u, lo.z ^ 0x80008000u, lo.w ^ 0x80008000u);
          *reinterpret_cast<uint4*>(pb + o + (8 + g) * 128) = hi;
          *reinterpret_cast<uint4*>(pb + PART + o + (8 + g) * 128) = lo;
          *reinterpret_cast<uint4*>(pb + o + g * 128) = nh;
          *reinterpret_cast<uint4*>(pb + PART + o + g * 128) = nl;
        }
      }
      fence_async_smem();
      tc_before();
      named_sync(BAR_MATH, NT);
      if constexpr (PR) {
        if (tid == 0 && !leader) mbar_arrive_peer(lead_bready);  // the leader's MMAs read our B half
        if (warp == 0) {
          tc_after();
          if (leader) {
            bwait_cl(&sm->bready, nq & 1);
            tc_after();
            for (int k = 0; k < NCH; ++k) {
              const uint32_t gc = g_cons + k;
              const int s = gc % NS;
              bwait(&sm->full[s], (gc / NS) & 1);
              bwait_cl(&sm->pfull[s], (gc / NS) & 1);
              if (p.trace && cid == 0 && rank == 0 && lane == 0 && gc < 64) p.trace[192 + gc] = clock64();
              tc_after();
              const uint32_t st = su32(ring + s * L::STAGE);
#pragma unroll
              for (int ai = 0; ai < 2; ++ai) {
                const uint64_t ah = sdesc(st + tile_off<true>(ai, 0, 0), 128, 256);
                const uint64_t al = sdesc(st + tile_off<true>(ai, 1, 0), 128, 256);
                const uint32_t bo = upb + 2 * k * LBOB + (ai ? 0 : JN / 8 * 128);  // B2 = [-Pi | Pr], B1 = [Pr | Pi]
                const uint64_t bh = sdesc(bo, LBOB, 128), bl = sdesc(bo + PART, LBOB, 128);
                const uint32_t acc = (k | ai) != 0;
                for (int rep = 0; rep < p.mma_reps; ++rep) {
                  mma2_w(tmem + T_Q, ah, bh, ID2, acc);
                  mma2_w(tmem + T_Q, ah, bl, ID2, 1);
                  mma2_w(tmem + T_Q, al, bh, ID2, 1);
                }
              }
              commit2_mc_w(&sm->empty[s], p.unicast ? pair_mask : ALL);
            }
            commit2_mc_w(&sm->q_full, pair_mask);
          } else {  // relay each landing of our row tile to the leader
            for (int k = 0; k < NCH; ++k) {
              const uint32_t gc = g_cons + k;
              const int s = gc % NS;
              bwait(&sm->full[s], (gc / NS) & 1);
              if (lane == 0) mbar_arrive_peer(lead_pfull + 8u * (uint32_t)s);
              __syncwarp();
            }
          }
          bwait_cl(&sm->q_full, nq & 1);
        } else if (warp == 1) {
          for (int k = 0; k < NCH; ++k) issue_next();
        }
        g_cons += NCH;
        named_sync(BAR_MATH, NT);
        ++nq;
        tc_after();
        if (remote) {  // our accumulator's rows of the peer's columns -> the peer
          float w[JN];
          tmem_ld<JN>(tQ, w);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < JN / 4; ++g)
            st_async_v4(peer_qx + 16u * (uint32_t)(g * 256 + qslot), w + 4 * g, peer_qxbar);
        }
      } else {
      if (warp == 0) {  // the whole warp issues (tcgen05 ops elect one lane)
        tc_after();
        for (int k = 0; k < NCH; ++k) {  // K-step k: Re A half, then Im A half
          const uint32_t gc = g_cons + k;
          const int s = gc % NS;
          if (p.spin) bwait<true>(&sm->full[s], (gc / NS) & 1);
          else bwait(&sm->full[s], (gc / NS) & 1);
          if (p.trace && cid == 0 && rank == 0 && lane == 0 && gc < 64) p.trace[192 + gc] = clock64();
          tc_after();
          if (!p.ss) {  // TMEM A operand: copy the chunk, then free its stage at once
#pragma unroll
            for (int ai = 0; ai < 2; ++ai) {
              const uint32_t st = su32(ring + s * CHUNK + ai * HALF);
              const uint32_t ta = tmem + T_A + 32 * ((2 * gc + ai) & 3);
#pragma unroll
              for (int x = 0; x < 4; ++x) tmem_cp_w(ta + 8 * x, sdesc(st + x * TILE, 128, 256));
            }
            if (p.unicast) commit_w(&sm->empty[s]);
            else commit_mc_w(&sm->empty[s], 0xFF);
          }
#pragma unroll
          for (int ai = 0; ai < 2; ++ai) {
            const uint32_t st = su32(ring + s * CHUNK + ai * HALF);
            const uint32_t ta = tmem + T_A + 32 * ((2 * gc + ai) & 3);
            const uint32_t bo = upb + 2 * k * LBOB + (ai ? 0 : JN / 8 * 128);  // B2 = [-Pi | Pr], B1 = [Pr | Pi]
            const uint64_t bh = sdesc(bo, LBOB, 128), bl = sdesc(bo + PART, LBOB, 128);
            const uint32_t acc = (k | ai) != 0;
            for (int rep = 0; rep < p.mma_reps; ++rep) {
              const uint32_t d0 = tmem + T_Q, d1 = tmem + T_Q + 2 * JN;  // row tiles interleaved
              if (p.ss) {
                mma_w(d0, sdesc(st + 0 * TILE, 128, 256), bh, ID, acc);
                mma_w(d1, sdesc(st + 1 * TILE, 128, 256), bh, ID, acc);
                mma_w(d0, sdesc(st + 0 * TILE, 128, 256), bl, ID, 1);
                mma_w(d1, sdesc(st + 1 * TILE, 128, 256), bl, ID, 1);
                mma_w(d0, sdesc(st + 2 * TILE, 128, 256), bh, ID, 1);
                mma_w(d1, sdesc(st + 3 * TILE, 128, 256), bh, ID, 1);
              } else {
                mma_ts_w(d0, ta + 0, bh, ID, acc);
                mma_ts_w(d1, ta + 8, bh, ID, acc);
                mma_ts_w(d0, ta + 0, bl, ID, 1);
                mma_ts_w(d1, ta + 8, bl, ID, 1);
                mma_ts_w(d0, ta + 16, bh, ID, 1);
                mma_ts_w(d1, ta + 24, bh, ID, 1);
              }
            }
          }
          if (p.ss) {
            if (p.unicast) commit_w(&sm->empty[s]);
            else commit_mc_w(&sm->empty[s], 0xFF);
          }
        }
        commit_w(&sm->q_full);
        bwait(&sm->q_full, nq & 1);
      } else if (warp == 1) {
        // producer (decoupled from the MMA issuer: a lane's bulk-copy issue can
        // stall it for hundreds of cycles): this product's remaining K-steps
        // and the next product's first NS, each once its stage is free
        for (int k = 0; k < NCH; ++k) issue_next();
      }
      g_cons += NCH;
      named_sync(BAR_MATH, NT);  // the other warps block in hardware until the products are done
      ++nq;
      tc_after();
      }
    };

    // Q = A P0 for the diagonal P0 (x0 = 0, b = I): column j of A times p_jj,
    // read from A in global memory (every other term of the product is an
    // exact zero) and stored in TMEM in the product's scaled units
    // (the CTA's 256 x 32 slab of A is read coalesced into the idle B-tile
    // region -- row stride 33 complex -- then each thread takes its row)
    auto first_q = [&]() {
      constexpr int SS = JN + 1;
      float2* slab = reinterpret_cast<float2*>(pb);
      const float4* a4 = reinterpret_cast<const float4*>(a + JN * cb);
      for (int f = tid; f < KU * (JN / 2); f += NT) {  // float4 f: row f / 16, columns 2 (f % 16), +1
        const int row = f / (JN / 2), c2 = f % (JN / 2);
        const float4 v = __ldg(a4 + (int64_t)row * (KU / 2) + c2);
        slab[row * SS + 2 * c2] = make_float2(v.x, v.y);
        slab[row * SS + 2 * c2 + 1] = make_float2(v.z, v.w);
      }
      named_sync(BAR_MATH, NT);
#pragma unroll
      for (int c0 = 0; c0 < JN; c0 += 8) {
        float sx[8], q8[8];
        lds8(sm->spx + c0, sx);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jg = JN * cb + c0 + i;
          const float2 av = slab[u * SS + c0 + i];
          const float p0 = use_c ? 1.0f / (sm->cdg[jg] * sa) : 1.0f;
          q8[i] = ((sa * (part ? av.y : av.x)) * p0) * sx[i];
        }
        if (remote) {  // PR: this thread's Q lives in the exchange buffer
          float4* qb = reinterpret_cast<float4*>(qxb);
          qb[(c0 / 4) * 256 + qslot] = make_float4(q8[0], q8[1], q8[2], q8[3]);
          qb[(c0 / 4 + 1) * 256 + qslot] = make_float4(q8[4], q8[5], q8[6], q8[7]);
        } else {
          tmem_st8(tQ + c0, q8);
        }
      }
      tmem_wait_st();
      named_sync(BAR_MATH, NT);  // the slab region is the next product's B tile
    };
    for (int t = 1; t <= p.T; ++t) {
      stamp();
      scale(P);
      stamp();
      if (t == 1) first_q();
      else product(P);
      stamp();
      const float qs = (use_c && !textbook) ? icr : 1.0f;  // Algorithm 1: z = C^-1 P m
      const float4* qb = reinterpret_cast<const float4*>(qxb);
      if (remote) {  // PR: Q of this thread's rows was computed by the peer
        if (t > 1) bwait_cl(&sm->qx, (nq - 1) & 1);
#pragma unroll
        for (int g = 0; g < JN / 4; ++g) {
          const float4 x = qb[g * 256 + qslot];
          A[4 * g] = x.x; A[4 * g + 1] = x.y; A[4 * g + 2] = x.z; A[4 * g + 3] = x.w;
        }
      } else {
        tmem_ld<JN>(tQ, A);
        tmem_wait_ld();
      }
      // curvature m^H z per column (linsolve.py:276)
#pragma unroll
      for (int c0 = 0; c0 < JN; c0 += 8) {
        float sy[8];
        lds8(sm->spy + c0, sy);
#pragma unroll
        for (int i = 0; i < 8; ++i) A[c0 + i] = P[c0 + i] * ((A[c0 + i] * sy[i]) * qs);
      }
      col_partials(A, sm, warp);
      named_sync(BAR_MATH, NT);
      if (tid < JN) {  // alpha_j, NotHpd (linsolve.py:277-280)
        const float curv = col_total(sm, tid);
        const float rzj = sm->rzs[tid];
        const bool act = rzj > 0.0f;
        if (curv <= 0.0f && act) sm->not_hpd = 1;
        sm->coef[0][tid] = act ? rzj / (curv > 0.0f ? curv : 1.0f) : 0.0f;
      }
      named_sync(BAR_MATH, NT);
      // w += alpha m, r -= alpha Pm, rz partials (linsolve.py:281-284)
#pragma unroll
      for (int c0 = 0; c0 < JN; c0 += 8) {
        float qv[8], rv[8], xv[8], al8[8], sy[8];
        if (remote) {
          const float4 x = qb[(c0 / 4) * 256 + qslot], y = qb[(c0 / 4 + 1) * 256 + qslot];
          qv[0] = x.x; qv[1] = x.y; qv[2] = x.z; qv[3] = x.w; qv[4] = y.x; qv[5] = y.y; qv[6] = y.z; qv[7] = y.w;
        } else {
          tmem_ld8(tQ + c0, qv);
        }
        tmem_ld8(tR + c0, rv);
        tmem_ld8(tX + c0, xv);
        lds8(sm->coef[0] + c0, al8);
        lds8(sm->spy + c0, sy);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float al = al8[i];
          xv[i] = xv[i] + al * P[c0 + i];
          rv[i] = rv[i] - al * ((qv[i] * sy[i]) * qs);
          const float z = textbook ? rv[i] * icr : rv[i];
          A[c0 + i] = rv[i] * z;
        }
        tmem_st8(tR + c0, rv);
        tmem_st8(tX + c0, xv);
      }
      col_partials(A, sm, warp);
      tmem_wait_st();
      stamp();
      named_sync(BAR_MATH, NT);
      if (tid < JN) {  // beta_j, rz update (linsolve.py:284-288)
        const float rn = col_total(sm, tid);
        const float rzj = sm->rzs[tid];
        sm->coef[1][tid] = rzj > 0.0f ? rn / rzj : 0.0f;
        sm->rzs[tid] = rn;
      }
      named_sync(BAR_MATH, NT);
      // m = z + beta m
#pragma unroll
      for (int c0 = 0; c0 < JN; c0 += 8) {
        float rv[8], be8[8];
        tmem_ld8(tR + c0, rv);
        lds8(sm->coef[1] + c0, be8);
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
    stamp();
    tmem_ld<JN>(tX, P);
    tmem_ld<JN>(tR, A);
    tmem_wait_ld();
    stamp();
    double fro = 0.0;
    const double xsa = alpha * (double)sa;
    const float crr = (use_c && !textbook) ? cr : 1.0f;
    double rs = 0.0;  // this thread's part of sum_j |GX_uj|^2 over the CTA's columns
    float gd = 0.0f;  // its part of GX_uu when column u is the CTA's
#pragma unroll
    for (int jj = 0; jj < JN; ++jj) {
      const int jg = JN * cb + jj;
      const float e = (part == 0 && u == jg) ? 1.0f : 0.0f;
      const float ax = e - crr * A[jj];
      const float g = (float)((double)ax - xsa * (double)P[jj]);
      A[jj] = g;
      fro += (double)(P[jj] * sa) * (double)g;  // Re tr(X^H GX)
      rs += (double)(g * g);
      if (u == jg) gd = g;
    }
    // SINR inputs instead of GX itself (metrics.py:35-58 needs |B_kk|^2 and the
    // row sums of |B_kj|^2 only): 16 KiB per realization instead of 512 KiB
    if (p.rsq) {
      p.rsq[((b * C + cb) * 2 + part) * KU + u] = rs;
      if ((unsigned)(u - JN * cb) < (unsigned)JN) reinterpret_cast<float*>(p.gdiag + b * KU + u)[part] = gd;
    }
    // ---- outputs staged in the (idle: every chunk of this realization has
    // landed and been consumed) ring as [user][column][re, im] with an odd row
    // stride (conflict-free), then written as coalesced 256-B row segments
    constexpr int SR = 2 * JN + 1;
    float* stg = reinterpret_cast<float*>(ring);
    stamp();
#pragma unroll 1
    for (int pass = 0; pass < (p.rsq ? 1 : 2); ++pass) {
#pragma unroll
      for (int jj = 0; jj < JN; ++jj) stg[u * SR + 2 * jj + part] = pass == 0 ? P[jj] * sa : A[jj];
      named_sync(BAR_MATH, NT);
      float* out = reinterpret_cast<float*>((pass == 0 ? p.X : p.GX) + b * (int64_t)KU * KU + JN * cb);
      for (int row = warp; row < KU; row += NT / 32) {
        out[(int64_t)row * 2 * KU + lane] = stg[row * SR + lane];
        out[(int64_t)row * 2 * KU + 32 + lane] = stg[row * SR + 32 + lane];
      }
      named_sync(BAR_MATH, NT);
      if (pass == 0) stamp();
    }
    if (p.xmax) {  // per-column max |X| for the W kernel's row scales (saves it a pass over X)
#pragma unroll
      for (int jj = 0; jj < JN; ++jj) A[jj] = fabsf(P[jj] * sa);
      col_partials<true>(A, sm, warp);
      named_sync(BAR_MATH, NT);
      if (tid < JN) p.xmax[b * KU + JN * cb + tid] = col_total<true>(sm, tid);
      named_sync(BAR_MATH, NT);
    }
    stamp();
    fro = warp_sum(fro);
    if (lane == 0) sm->dred[warp] = fro;
    named_sync(BAR_MATH, NT);
    if (tid == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 16; ++w) s += sm->dred[w];
      p.part[C * b + cb] = s;
      if (zsum > 0.0f) {
        if (cb == 0) p.status[b] = XL_STATUS_SPLITTING;
      } else if (sm->not_hpd) {
        atomicCAS(reinterpret_cast<int*>(p.status + b), 0, XL_STATUS_NOT_HPD);
      }
    }
  }
  tc_before();
  cluster_sync();  // no multicast may target an exited CTA
  if (warp == 0) {
    tc_after();
    tmem_free512_g<PR>(tmem);
  }
}
}  // namespace pc

// ============================================================ W, CTA pairs ===
// lk_w_kernel as cta_group::2 pairs (XL_LK_W2=1): output blocks t = 2p, 2p + 1
// of one realization form a cluster of two and multiply as one M = 256 MMA
// (each CTA's A = its block's X rows, written into its own TMEM with
// tcgen05.st), N = 64 antennas split 32 / 32: each CTA lands and converts only
// its 32-antenna half of every H box and the pair's tensor cores read both
// halves, so per CTA and box the shared-memory port moves 36 KiB instead of 72.
// The follower's converter warps signal the leader's MMA issuer directly
// (mbarrier.arrive.release.cluster); they never hold outstanding global
// stores (a dedicated epilogue warpgroup drains TMEM and writes W), which made
// that release cost a third of the kernel in the first pair version.
namespace wk2 {
using wk::CHA;
using wk::BU;
using wk::TPR;
using wk::T_AH;
using wk::T_AL;
using wk::T_ACC;
constexpr int W_PROD = 0, W_MMA = 1, W_CONV0 = 2, NCONV = 8, W_EPI0 = W_CONV0 + NCONV, NEPI = 4;
constexpr int NT = 32 * (W_EPI0 + NEPI);
constexpr int HB = (CHA / 2) * 2 * BU * 4;  // 8 KiB: this CTA's 32 antennas of a box
constexpr int NS = 20;                      // ring depth (160 KiB in flight)
constexpr int SMALL = 2048;
constexpr int SMEM = NS * HB + SMALL;
static_assert(SMEM <= 227 * 1024, "lk W2 smem");
constexpr uint32_t ID2 = idesc(256, CHA, 0, 0);

struct Small {
  uint64_t full[NS], conv[NS], freed[NS];
  uint64_t acc_full[2], acc_free[2], pacc_free[2];
  uint32_t tmem_slot;
  float rmax[4][64];
  float sx[64];
};
static_assert(sizeof(Small) <= SMALL, "W2 small");

__device__ __forceinline__ void tmem_st16u(uint32_t ta, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__global__ void __launch_bounds__(NT, 1) lk_w2_kernel(const __grid_constant__ CUtensorMap hmap, int M,
                                                      const unsigned* __restrict__ zmax, const float2* __restrict__ X,
                                                      const double* __restrict__ beta, float* __restrict__ W,
                                                      float* __restrict__ F, const float* __restrict__ xmax) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small* sm = reinterpret_cast<Small*>(smem + NS * HB);
  const int64_t b = blockIdx.x / TPR;
  const int t = blockIdx.x % TPR;
  const uint32_t pr = cluster_rank();  // == t & 1
  const bool leader = pr == 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntile = M / CHA, nbox = ntile * (KU / BU);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->conv[s], 2 * 4);  // leader: the 4 converter warps of this box in each CTA
      mbar_init(&sm->freed[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&sm->acc_full[j], 1);
      mbar_init(&sm->acc_free[j], NEPI);  // the local epilogue warps
      mbar_init(&sm->pacc_free[j], 1);    // leader: the follower's epilogue (relayed)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) pc::tmem_alloc512_g<true>(&sm->tmem_slot);
  const float2* Xb = X + b * (int64_t)KU * KU;
  // ---- per-user scale sx[j'] = 2^e, max |X_:j'| sx < 2^14
  if (xmax) {  // the solver's per-column max |X|
    if (tid < 64) sm->sx[tid] = pow2_scale(xmax[b * KU + 64 * t + tid], 14);
    tc_before();
    __syncthreads();
    tc_after();
  } else {
    if (tid < 256) {
      const int jl = tid & 63, part = tid >> 6;
      float m = 0.0f;
#pragma unroll 8
      for (int i = 64 * part; i < 64 * part + 64; ++i) {
        const float2 x = __ldg(Xb + (int64_t)i * KU + 64 * t + jl);
        m = fmaxf(m, fmaxf(fabsf(x.x), fabsf(x.y)));
      }
      sm->rmax[part][jl] = m;
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (tid < 64)
      sm->sx[tid] = pow2_scale(fmaxf(fmaxf(sm->rmax[0][tid], sm->rmax[1][tid]), fmaxf(sm->rmax[2][tid], sm->rmax[3][tid])), 14);
    __syncthreads();
  }
  const uint32_t tmem = sm->tmem_slot;
  // ---- A hi / lo straight into TMEM (lane = output row r, column = two input
  // users): converter warp cw writes its lane quadrant, users [128 h, +128)
  if (warp >= W_CONV0 && warp < W_EPI0) {
    const int cw = warp - W_CONV0, q = warp & 3, h = cw >> 2;
    const int r = 32 * q + lane, jl = r >> 1;
    const bool odd = r & 1;
    const float sc = sm->sx[jl];
    const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {  // 32 input users per step
      const int i0 = 128 * h + 32 * c;
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float2 x0 = __ldg(Xb + (int64_t)(i0 + 2 * e) * KU + 64 * t + jl);
        const float2 x1 = __ldg(Xb + (int64_t)(i0 + 2 * e + 1) * KU + 64 * t + jl);
        split2((odd ? x0.y : x0.x) * sc, (odd ? x1.y : x1.x) * sc, hi[e], lo[e]);
      }
      tmem_st16u(ta + T_AH + i0 / 2, hi);
      tmem_st16u(ta + T_AL + i0 / 2, lo);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_before();
  cluster_sync();  // both CTAs' A rows are in TMEM, every barrier initialised
  tc_after();

  if (warp == W_PROD) {
    constexpr int NL = 8;
    if (lane < NL) {
      const int y0 = (int)(b * M) + (CHA / 2) * (int)pr;
      for (int g = lane; g < nbox; g += NL) {
        const int s = g % NS, tt = g / (KU / BU), kb = g % (KU / BU);
        if (g >= NS) bwait<true>(&sm->freed[s], ((g / NS) - 1) & 1);
        mbar_expect_tx(&sm->full[s], HB);
        tma2d(ring + s * HB, &hmap, 2 * BU * kb, y0 + CHA * tt, &sm->full[s]);
      }
    }
  } else if (warp == W_MMA) {
    if (leader) {
      for (int g = 0; g < nbox; ++g) {
        const int s = g % NS, tt = g / (KU / BU), kb = g % (KU / BU);
        if (kb == 0 && tt >= 2) {
          bwait(&sm->acc_free[tt & 1], ((tt >> 1) - 1) & 1);
          pc::bwait_cl(&sm->pacc_free[tt & 1], ((tt >> 1) - 1) & 1);
        }
        pc::bwait_cl(&sm->conv[s], (g / NS) & 1);
        tc_after();
        const uint32_t st = su32(ring + s * HB);
        const uint32_t d1 = tmem + T_ACC + 128 * (tt & 1), d2 = d1 + CHA;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int sk = 2 * kb + ks;
          const uint32_t ah = tmem + T_AH + 8 * sk, al = tmem + T_AL + 8 * sk;
          const uint64_t brh = sdesc(st + 256 * ks, 128, 2048), brl = sdesc(st + 1024 + 256 * ks, 128, 2048);
          const uint64_t bih = sdesc(st + 512 + 256 * ks, 128, 2048), bil = sdesc(st + 1536 + 256 * ks, 128, 2048);
          const uint32_t acc = (kb | ks) != 0;
          mma2_ts_w(d1, ah, brh, ID2, acc);
          mma2_ts_w(d1, ah, brl, ID2, 1);
          mma2_ts_w(d1, al, brh, ID2, 1);
          mma2_ts_w(d2, ah, bih, ID2, acc);
          mma2_ts_w(d2, ah, bil, ID2, 1);
          mma2_ts_w(d2, al, bih, ID2, 1);
        }
        commit2_mc_w(&sm->freed[s], 3);
        if (kb == KU / BU - 1) commit2_mc_w(&sm->acc_full[tt & 1], 3);
      }
    } else if (lane == 0) {  // relay: the follower's drain of tile tt - 2 -> the leader
      const uint32_t lead_pfree = mapa_u32(su32(&sm->pacc_free[0]), 0);
      for (int tt = 2; tt < ntile; ++tt) {
        bwait(&sm->acc_free[tt & 1], ((tt >> 1) - 1) & 1);
        mbar_arrive_peer(lead_pfree + 8u * (uint32_t)(tt & 1));
      }
    }
  } else if (warp < W_EPI0) {  // converters: 8-antenna group grp of boxes g % 2 == par
    const int cw = warp - W_CONV0;
    const int grp = cw & 3, par = cw >> 2;
    const float sz = pow2_scale(__uint_as_float(zmax[b]), 11);
    const int crow = lane >> 2, pair = lane & 3;
    const uint32_t conv_addr = mapa_u32(su32(&sm->conv[0]), 0);
    for (int g = par; g < nbox; g += 2) {
      const int s = g % NS;
      bwait(&sm->full[s], (g / NS) & 1);
      uint8_t* gb = ring + s * HB + grp * 2048;  // 8 antennas x 64 components
      float4 v[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int c = (it + crow) & 3;
        v[it] = *reinterpret_cast<const float4*>(gb + crow * 256 + 64 * c + 16 * pair);
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int c = (it + crow) & 3;
        uint32_t hr, lr, hi_, li_;
        split2(v[it].x * sz, v[it].z * sz, hr, lr);
        split2(v[it].y * sz, v[it].w * sz, hi_, li_);
        const int o = crow * 16 + 4 * pair;
        *reinterpret_cast<uint32_t*>(gb + 128 * c + o) = hr;
        *reinterpret_cast<uint32_t*>(gb + 1024 + 128 * c + o) = lr;
        *reinterpret_cast<uint32_t*>(gb + 128 * (4 + c) + o) = hi_;
        *reinterpret_cast<uint32_t*>(gb + 1024 + 128 * (4 + c) + o) = li_;
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sm->conv[s]);
        else mbar_arrive_peer(conv_addr + 8u * (uint32_t)s);
      }
    }
  } else {  // epilogue warpgroup: lane quadrant q, all 64 antennas of a tile in two halves
    const int q = warp & 3;
    const int r = 32 * q + lane;  // output row (TMEM lane)
    const bool odd = r & 1;
    const int col = 128 * t + r;
    const double bt = beta[b];
    const float srow = sm->sx[r >> 1];
    const float sz = pow2_scale(__uint_as_float(zmax[b]), 11);
    const float wmul = (float)(bt / ((double)srow * (double)sz));
    const float fmul = 1.0f / (srow * sz);
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + T_ACC;
    for (int tt = 0; tt < ntile; ++tt) {
      const int jb = tt & 1;
      pc::bwait_cl(&sm->acc_full[jb], (tt >> 1) & 1);
      tc_after();
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        float v[32], u[32];
        tmem_ld16(tq + 128 * jb + 32 * hh, v);
        tmem_ld16(tq + 128 * jb + 32 * hh + 16, v + 16);
        tmem_ld16(tq + 128 * jb + CHA + 32 * hh, u);
        tmem_ld16(tq + 128 * jb + CHA + 32 * hh + 16, u + 16);
        tmem_wait_ld();
        if (hh == 1) {
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm->acc_free[jb]);
        }
#pragma unroll
        for (int n = 0; n < 32; ++n) {
          const float o2 = __shfl_xor_sync(0xffffffffu, u[n], 1);
          v[n] = odd ? v[n] + o2 : v[n] - o2;
        }
        const int64_t n0 = (int64_t)tt * CHA + 32 * hh;
        float* wp = W + (b * (int64_t)M + n0) * NC + col;
#pragma unroll
        for (int n = 0; n < 32; ++n) __stcs(wp + (int64_t)n * NC, v[n] * wmul);
        if (F) {
          float* fp = F + (b * (int64_t)M + n0) * NC + col;
#pragma unroll
          for (int n = 0; n < 32; ++n) __stcs(fp + (int64_t)n * NC, v[n] * fmul);
        }
      }
    }
  }
  tc_before();
  cluster_sync();  // no remote arrive / multicast commit targets an exited CTA
  if (warp == W_MMA) {
    tc_after();
    pc::tmem_free512_g<true>(tmem);
  }
}
}  // namespace wk2

// ========================================================= Gram, CTA pairs ===
// lk_gram_kernel as cta_group::2 pairs: the 512 x 512 real Gram's upper
// triangle as three 256 x 256 super-tiles (0,0), (0,1), (1,1), one CTA pair
// each (six CTAs per realization).  Pair CTA v of super-tile (I, J) supplies
// the M rows of 64-user block 2I + v and the N half of block 2J + v: on the
// diagonal super-tiles that is one block (landed and converted once, used as
// both operands), off the diagonal two.  Per CTA and 32-antenna chunk the
// shared-memory port moves 96-144 KiB instead of 144-216 KiB (a converted block
// feeds an M = 256 x N = 256 MMA), for 20% more MMA work (the lower quarters
// of the diagonal super-tiles).  The follower's converters signal the leader's
// MMA issuer with CTA-scope peer arrives; each CTA keeps its own split scale
// (first non-zero chunk) and the epilogue unscales column half k by the scale
// of the CTA that supplied it.
namespace gram2 {
using gram::CH;
using gram::BLK;
using gram::SGL;
using gram::NCONV;
using gram::W_PROD;
using gram::W_MMA;
using gram::W_CONV0;
using gram::NT;
using gram::BAR_CONV;
constexpr int TPR = 6;
constexpr int NS = 4;
constexpr int SB = 2 * SGL;  // 32 KiB: at most two single blocks per chunk
constexpr int SMALL = 1024;
constexpr int SMEM = NS * SB + SMALL;
static_assert(SMEM <= 227 * 1024, "lk gram2 smem");
constexpr uint32_t ID2 = idesc(256, 2 * BLK, 1, 1);
constexpr int SG = 8 * BLK * 4;  // one 8-antenna group of a single block (4 KiB raw == hi + lo)

struct Small {
  uint64_t full[NS], conv[NS], freed[NS];
  uint64_t done;
  uint32_t tmem_slot;
  float sz;
  float rmax[NCONV];
};
static_assert(sizeof(Small) <= SMALL, "gram2 small");

__global__ void __launch_bounds__(NT, 1) lk_gram2_kernel(const __grid_constant__ CUtensorMap smap, int M,
                                                         float* __restrict__ szv, float2* __restrict__ A, double xi,
                                                         const double* __restrict__ xi_b, int* __restrict__ rflag,
                                                         unsigned* __restrict__ zmax, int fixup) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Small* sm = reinterpret_cast<Small*>(smem + NS * SB);
  const int64_t b = blockIdx.x / TPR;
  const int st_idx = (blockIdx.x % TPR) >> 1;  // super-tile 0: (0,0), 1: (0,1), 2: (1,1)
  if (fixup && rflag[b] == 0) return;           // both CTAs of the pair share b
  const uint32_t v = cluster_rank();
  const bool leader = v == 0;
  const int SI = st_idx == 2 ? 1 : 0, SJ = st_idx == 0 ? 0 : 1;
  const bool diag = SI == SJ;
  const int rowblk = 2 * SI + (int)v, colblk = 2 * SJ + (int)v;
  const int nbx = diag ? 1 : 2;  // singles per chunk: [rowblk] or [rowblk, colblk]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = M / CH;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->conv[s], 2 * NCONV);  // leader: every converter warp of both CTAs
      mbar_init(&sm->freed[s], 1);
    }
    mbar_init(&sm->done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) pc::tmem_alloc512_g<true>(&sm->tmem_slot);
  tc_before();
  __syncthreads();
  tc_after();
  cluster_sync();  // barriers initialised in both CTAs before any peer arrive / multicast commit
  const uint32_t tmem = sm->tmem_slot;

  float sz = fixup ? szv[b] : 1.0f;
  if (warp == W_PROD) {
    if (lane < nbx) {
      const int y0 = (int)(b * M);
      const int blk = lane == 0 ? rowblk : colblk;
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        if (c >= NS) bwait<true>(&sm->freed[s], ((c / NS) - 1) & 1);
        if (lane == 0) mbar_expect_tx(&sm->full[s], nbx * SGL);
        tma2d(ring + s * SB + lane * SGL, &smap, BLK * blk, y0 + c * CH, &sm->full[s]);
      }
    }
  } else if (warp == W_MMA) {
    if (leader) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        pc::bwait_cl(&sm->conv[s], (c / NS) & 1);
        tc_after();
        const uint32_t sa = su32(ring + s * SB), sbb = sa + (diag ? 0 : SGL);
#pragma unroll
        for (int ks = 0; ks < CH / 16; ++ks) {
          const uint32_t acc = (c | ks) != 0;
          const uint64_t ah = sdesc(sa + 2 * ks * SG, SG, 128), al = sdesc(sa + 2 * ks * SG + SG / 2, SG, 128);
          const uint64_t bh = sdesc(sbb + 2 * ks * SG, SG, 128), bl = sdesc(sbb + 2 * ks * SG + SG / 2, SG, 128);
          mma2_w(tmem, ah, bh, ID2, acc);
          mma2_w(tmem, ah, bl, ID2, 1);
          mma2_w(tmem, al, bh, ID2, 1);
        }
        commit2_mc_w(&sm->freed[s], 3);
      }
      commit2_mc_w(&sm->done, 3);
    }
  } else {
    const int cw = warp - W_CONV0;
    const bool active = cw < 4 * nbx;  // group cw & 3 of single cw >> 2
    bool have = fixup != 0, over = false;
    float zm = 0.0f;
    const uint32_t conv_addr = mapa_u32(su32(&sm->conv[0]), 0);
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      bwait(&sm->full[s], (c / NS) & 1);
      uint8_t* sg = ring + s * SB + (cw >> 2) * SGL + (cw & 3) * SG;
      float4 vs[8];
      float gm = active ? gram::load8(sg, BLK * 4, lane, 0, vs) : 0.0f;
      zm = fmaxf(zm, gm);
      if (!have) {  // until the first non-zero chunk: max over the converter warps
        gm = warp_max(gm);
        if (lane == 0) sm->rmax[cw] = gm;
        named_sync(BAR_CONV, 32 * NCONV);
        float mx = sm->rmax[0];
#pragma unroll
        for (int w = 1; w < NCONV; ++w) mx = fmaxf(mx, sm->rmax[w]);
        named_sync(BAR_CONV, 32 * NCONV);
        if (mx > 0.0f) {
          sz = pow2_scale(mx, 7);
          have = true;
        }
      }
      over |= !(gm * sz < RANGE_MAX);
      __syncwarp();
      if (active) gram::store8(sg, SG / 2, lane, 0, vs, sz);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sm->conv[s]);
        else mbar_arrive_peer(conv_addr + 8u * (uint32_t)s);
      }
    }
    over = __any_sync(0xffffffffu, over);
    zm = warp_max(zm);
    if (!fixup && over && lane == 0) rflag[b] = 1;
    if (lane == 0 && zm > 0.0f) atomicMax(zmax + b, __float_as_uint(zm));
    if (tid == 32 * W_CONV0) sm->sz = sz;
  }
  tc_before();
  cluster_sync();  // both CTAs' scales are published
  tc_after();
  if (warp >= W_CONV0) {
    // ---- epilogue: column half k of the accumulator is tile (rowblk, 2 SJ + k),
    // supplied by CTA k; the upper-triangle tiles are written with their
    // conjugate mirror (Hermitian by construction), the lower one skipped
    float szk[2];
    {
      float peer_sz;
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(peer_sz) : "r"(mapa_u32(su32(&sm->sz), v ^ 1u)));
      szk[v] = sm->sz;
      szk[v ^ 1u] = peer_sz;
    }
    pc::bwait_cl(&sm->done, 0);
    tc_after();
    const int cw = warp - W_CONV0;
    const int q = warp & 3, p = cw >> 2;
    const int r = 32 * q + lane;
    const double xi_v = xi_b ? xi_b[b] : xi;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const bool odd = lane & 1;
    float2* Ab = A + b * (int64_t)KU * KU;
    const float isz_row = 1.0f / sm->sz;
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
      const int I = rowblk, J = 2 * SJ + k;
      if (I > J) continue;
      const float un = isz_row / szk[k];
      const int i = 64 * I + (r >> 1);
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float vv[16];
        tmem_ld16(tl + 128 * k + 64 * p + c0, vv);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float g0 = vv[e] * un, g1 = vv[e + 1] * un;
          const float p0 = __shfl_xor_sync(0xffffffffu, g0, 1), p1 = __shfl_xor_sync(0xffffffffu, g1, 1);
          float re = odd ? (p0 + g1) : (g0 + p1);
          const float im = odd ? (p1 - g0) : (g1 - p0);
          const int j = 64 * J + ((64 * p + c0 + e) >> 1);
          if (i == j) {
            if (!odd) Ab[(int64_t)i * KU + j] = make_float2((float)((double)re + xi_v), 0.0f);
          } else if (i < j) {
            if (!odd) Ab[(int64_t)i * KU + j] = make_float2(re, im);
            else Ab[(int64_t)j * KU + i] = make_float2(re, -im);
          }
        }
      }
    }
  }
  tc_before();
  cluster_sync();  // no peer arrive / multicast commit targets an exited CTA
  if (warp == W_MMA) {
    tc_after();
    pc::tmem_free512_g<true>(tmem);
  }
}
}  // namespace gram2

// ------------------------------------------------------------------ SINR ----
// gamma_k = |B_kk|^2 / (sum_j |B_kj|^2 - |B_kk|^2 + sigma2), B = beta GX
// (coupling_matrix + sinr_eq9, metrics.py:35-58) from the solver's per-block
// row sums and diagonal; sum-SE in user order (as sinr_kernel).
__global__ void __launch_bounds__(KU) lk_sinr_kernel(const double* __restrict__ rsq, const float2* __restrict__ gd,
                                                     const double* __restrict__ beta, double sigma2,
                                                     double* __restrict__ gamma, double* __restrict__ sum_se) {
  const int64_t b = blockIdx.x;
  const int k = threadIdx.x;
  __shared__ double sse[KU];
  const double s2 = beta[b] * beta[b];
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < 2 * pc::C; ++q) tot += rsq[(b * 2 * pc::C + q) * KU + k];
  tot *= s2;
  const float2 d = gd[b * KU + k];
  const double sig = (double)cabs2(d) * s2;
  const double g = sig / ((tot - sig) + sigma2);
  const double se = log2(1.0 + g);
  if (gamma) gamma[b * KU + k] = g;
  sse[k] = se;
  __syncthreads();
  if (k == 0) {
    double t = 0.0;
    for (int i = 0; i < KU; ++i) t += sse[i];
    sum_se[b] = t;
  }
}

// ------------------------------------------------------------------ host ----
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  }
  return fn;
}

// H[B][M][K] complex64 as a 2-D fp32 tensor [B M rows][2K floats], box {bx, by}
static int make_hmap(CUtensorMap* map, const void* H, int64_t B, int M, int bx, int by) {
  EncodeTiled enc = encoder();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return XL_ERR_CUDA; }
  const cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)(B * M)};
  const cuuint64_t strides[1] = {(cuuint64_t)NC * 4};
  const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(H), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("tensor map encode failed (%d)", (int)r); return XL_ERR_CUDA; }
  return XL_SUCCESS;
}

}  // namespace lk

bool lk_supported(int dtype, int M, int K) {
  if (dtype != XL_C64 || K != lk::KU || M < 64 || M % 64 != 0) return false;
  const char* e = getenv("XL_LARGE_K_256");  // "library": the split-operand library GEMM path (A/B, tests)
  return !(e && e[0] == 'l');
}

// the pair-MMA solver (PR) unless XL_LK_PAIR=0 (A/B, tests)
static bool lk_pair() {
  const char* e = getenv("XL_LK_PAIR");
  return !(e && e[0] == '0');
}

template <bool PR>
static int lk_clusters() {
  static int n = 0;
  if (n == 0) {
    auto kern = lk::pc::lk_pcg_kernel<PR>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lk::pc::smem_bytes<PR>());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lk::pc::cl_size<PR>() * 16, 1, 1);
    cfg.blockDim = dim3(lk::pc::NT, 1, 1);
    cfg.dynamicSmemBytes = lk::pc::smem_bytes<PR>();
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = lk::pc::cl_size<PR>();
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c < 1) {
      cudaGetLastError();
      c = 16;
    }
    n = c;
  }
  return n;
}

// scratch: sz[B] floats, range flags[B] ints (Gram), the same for W, and the
// cluster solver's A'' slots
size_t lk_ws_bytes(int64_t B) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return 4 * al((size_t)B * 4) + (size_t)lk::pc::MAX_SLOTS * lk::pc::SLOT_BYTES;
}

LkScratch lk_scratch(void* ws, int64_t B) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char* p = (char*)ws;
  LkScratch r;
  r.sz = (float*)p;
  r.rflag = (int*)(p + al((size_t)B * 4));
  r.zmax = (unsigned*)(p + 2 * al((size_t)B * 4));
  r.slots = (uint8_t*)(p + 4 * al((size_t)B * 4));
  return r;
}

int lk_gram(const void* H, int64_t B, int M, double xi, const double* xi_b, void* A, float* sz, int* rflag,
            unsigned* zmax, cudaStream_t st) {
  using namespace lk;
  CUtensorMap pmap, smap;
  if (int e = make_hmap(&pmap, H, B, M, 2 * gram::BLK, gram::CH)) return e;
  if (int e = make_hmap(&smap, H, B, M, gram::BLK, gram::CH)) return e;
  if (cudaMemsetAsync(rflag, 0, (size_t)B * sizeof(int), st) != cudaSuccess) return check_launch("lk flags");
  if (cudaMemsetAsync(zmax, 0, (size_t)B * sizeof(unsigned), st) != cudaSuccess) return check_launch("lk zmax init");
  const char* g2 = getenv("XL_LK_GRAM2");  // "0": the 5-CTA single-CTA-MMA Gram (A/B, tests)
  const bool pair = !(g2 && g2[0] == '0');
  auto launch = [&](int fixup) -> int {
    if (pair) {
      cudaFuncSetAttribute(gram2::lk_gram2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gram2::SMEM);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(gram2::TPR * B), 1, 1);
      cfg.blockDim = dim3(gram2::NT, 1, 1);
      cfg.dynamicSmemBytes = gram2::SMEM;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, gram2::lk_gram2_kernel, smap, M, sz, (float2*)A, xi, xi_b, rflag, zmax, fixup) !=
          cudaSuccess)
        return check_launch("lk gram2 launch");
      return check_launch(fixup ? "lk gram2 fixup" : "lk gram2");
    }
    cudaFuncSetAttribute(gram::lk_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gram::SMEM);
    gram::lk_gram_kernel<<<(unsigned)(gram::TPR * B), gram::NT, gram::SMEM, st>>>(pmap, smap, M, sz, (float2*)A, xi,
                                                                                 xi_b, rflag, zmax, fixup);
    return check_launch(fixup ? "lk gram fixup" : "lk gram");
  };
  if (int e = launch(0)) return e;
  lk_zmax_kernel<<<(unsigned)B, 512, 0, st>>>((const float4*)H, (int64_t)M * NC / 4, sz, rflag);
  if (int e = check_launch("lk zmax")) return e;
  return launch(1);
}

static long long* g_lk_trace = nullptr;
void lk_debug_trace(void* p) { g_lk_trace = (long long*)p; }

int lk_solve(int method, int variant, const void* A, int64_t B, int T, double xi, const double* xi_b, void* X,
             void* GX, double* part, int32_t* status, uint8_t* scratch, cudaStream_t st) {
  using namespace lk;
  const bool pair = lk_pair();
  int ncl = pair ? lk_clusters<true>() : lk_clusters<false>();
  if (ncl > pc::MAX_SLOTS) ncl = pc::MAX_SLOTS;
  if (ncl > (pair ? 2 * B : B)) ncl = (int)(pair ? 2 * B : B);
  const int cl = pair ? pc::cl_size<true>() : pc::cl_size<false>();
  const char* uc = getenv("XL_LK_UNICAST");
  // the GX buffer holds the SINR partials instead (lk_sinr): [B][8][2][K] doubles, then [B][K] float2
  double* rsq = (double*)GX;
  float2* gdiag = (float2*)(rsq + (size_t)B * pc::C * 2 * KU);
  float* xmax = lk_xmax(GX, B);
  pc::Params p{(const float2*)A, B, T, method, variant, xi, xi_b, (float2*)X, (float2*)GX, part, rsq, gdiag,
               xmax, status, scratch, g_lk_trace, (uc && uc[0] == '1') ? 1 : 0, 1, 1, 0};
  if (const char* sp = getenv("XL_LK_SPIN")) p.spin = sp[0] == '1';
  if (const char* ss = getenv("XL_LK_SS")) p.ss = ss[0] == '1';  // default 1: A from shared memory (measured faster than tcgen05.cp + TMEM)
  if (const char* mr = getenv("XL_LK_MMA_REPS")) p.mma_reps = atoi(mr) > 0 ? atoi(mr) : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cl * ncl), 1, 1);
  cfg.blockDim = dim3(pc::NT, 1, 1);
  cfg.dynamicSmemBytes = pair ? pc::smem_bytes<true>() : pc::smem_bytes<false>();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  auto kern = pair ? pc::lk_pcg_kernel<true> : pc::lk_pcg_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return check_launch("lk pcg launch");
  return check_launch("lk pcg");
}

float* lk_xmax(void* GX, int64_t B) {
  return (float*)((float2*)((double*)GX + (size_t)B * lk::pc::C * 2 * lk::KU) + (size_t)B * lk::KU);
}

int lk_sinr(const void* GX, const double* beta, int64_t B, double sigma2, double* gamma, double* sum_se,
            cudaStream_t st) {
  using namespace lk;
  const double* rsq = (const double*)GX;
  const float2* gdiag = (const float2*)(rsq + (size_t)B * pc::C * 2 * KU);
  lk_sinr_kernel<<<(unsigned)B, KU, 0, st>>>(rsq, gdiag, beta, sigma2, gamma, sum_se);
  return check_launch("lk sinr");
}

int lk_apply(const void* H, const void* X, const double* beta, int64_t B, int M, void* W, void* F,
             const unsigned* zmax, const float* xmax, cudaStream_t st) {  // zmax: from lk_gram; xmax: lk_solve or null
  using namespace lk;
  CUtensorMap map;
  const char* w2 = getenv("XL_LK_W2");  // "0": the single-CTA W kernel (A/B, tests)
  if (!(w2 && w2[0] == '0')) {  // CTA pairs: each CTA lands / converts half of every box
    if (int e = make_hmap(&map, H, B, M, 2 * wk::BU, wk::CHA / 2)) return e;
    cudaFuncSetAttribute(wk2::lk_w2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, wk2::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(wk::TPR * B), 1, 1);
    cfg.blockDim = dim3(wk2::NT, 1, 1);
    cfg.dynamicSmemBytes = wk2::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, wk2::lk_w2_kernel, map, M, zmax, (const float2*)X, beta, (float*)W, (float*)F, xmax) !=
        cudaSuccess)
      return check_launch("lk w2 launch");
    return check_launch("lk w2");
  }
  if (int e = make_hmap(&map, H, B, M, 2 * wk::BU, wk::CHA)) return e;
  cudaFuncSetAttribute(wk::lk_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, wk::SMEM);
  wk::lk_w_kernel<<<(unsigned)(wk::TPR * B), wk::NT, wk::SMEM, st>>>(map, M, zmax, (const float2*)X, beta, (float*)W,
                                                                     (float*)F);
  return check_launch("lk w");
}

}  // namespace xl
