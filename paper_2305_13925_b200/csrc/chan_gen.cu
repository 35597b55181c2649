// On-device channel-batch generation for the BASELINE model.
//
// Recipe (reference scenario.py:85-96, channel.py:33-53, geometry.py:169-180):
//   per user k: d ~ U[dmin, dmax], beta_dB = -35.3 - 37.6 log10 d,
//               gain = 10^(beta_dB/10) / beta_bar;
//   visibility: Bernoulli(p) per subarray, whole mask redrawn until >= 1 visible;
//   per visible subarray s: h = sqrt(gain) * R^{1/2} g,  g ~ CN(0, I_Ms).
// Random stream: Philox4x32-10, key = seed, counter = (j, k | purpose<<24,
// b_lo, b_hi) -- identical to oracle/xlmimo_oracle.py::generate_channels, so
// realization b is the same on any GPU count / chunking.
//
// chan_real_kernel (S * K <= 2^14, every BASELINE config): one CTA per
// realization draws the users' gains / visibility once and walks the
// subarrays.  chan_kernel (larger S * K): one CTA per (realization, subarray),
// every CTA re-deriving the users' gains / visibility.  Both write H rows
// coalesced (row m = s*Ms + i holds all K users contiguously), no workspace.
#include <math.h>

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {

enum { PURPOSE_DIST = 0, PURPOSE_VIS = 1, PURPOSE_FADE = 2 };
constexpr int MAX_VIS_ATTEMPTS = 4096;
constexpr int KCH = 64;  // users per smem chunk

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u01(uint32_t x) { return ((double)x + 0.5) * (1.0 / 4294967296.0); }

template <typename R>
__global__ void __launch_bounds__(256)
chan_kernel(uint64_t seed, int64_t first, int S, int Ms, int K, double p,
            const double* __restrict__ Rsqrt, double beta_bar, double dmin, double dmax,
            cplx<R>* __restrict__ H, int32_t* __restrict__ status) {
  using C = cplx<R>;
  const int64_t bl = blockIdx.x;           // local realization
  const int s = blockIdx.y;                // subarray
  const uint64_t bg = (uint64_t)(first + bl);
  const uint32_t b_lo = (uint32_t)bg, b_hi = (uint32_t)(bg >> 32);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int M = S * Ms;
  extern __shared__ double smem[];
  R* rs = (R*)smem;                        // Ms x Ms
  R* amp = rs + Ms * Ms;                   // K (0 when subarray s invisible)
  C* g = (C*)(amp + ((K + 1) & ~1));       // Ms x KCH
  const int tid = threadIdx.x;
  for (int e = tid; e < Ms * Ms; e += blockDim.x) rs[e] = (R)Rsqrt[e];
  const int nq = (S + 3) / 4;
  for (int k = tid; k < K; k += blockDim.x) {
    uint4 x = philox4x32_10(make_uint4(0u, (uint32_t)k | (PURPOSE_DIST << 24), b_lo, b_hi), k0, k1);
    double d = dmin + (dmax - dmin) * u01(x.x);
    double bdb = -35.3 - 37.6 * log10(d);
    double gain = pow(10.0, bdb / 10.0) / beta_bar;
    // visibility of subarray s in the first attempt with >= 1 visible subarray
    bool vis_s = false, found = false;
    for (int att = 0; att < MAX_VIS_ATTEMPTS && !found; ++att) {
      bool any = false;
      for (int q = 0; q < nq; ++q) {
        uint4 y = philox4x32_10(make_uint4((uint32_t)(att * nq + q), (uint32_t)k | (PURPOSE_VIS << 24), b_lo, b_hi), k0, k1);
        uint32_t w[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int ss = 4 * q + e;
          if (ss < S) {
            bool v = u01(w[e]) < p;
            any |= v;
            if (ss == s) vis_s = v;
          }
        }
      }
      found = any;
    }
    if (!found && s == 0) status[bl] = XL_STATUS_NO_VISIBLE;
    amp[k] = (found && vis_s) ? (R)sqrt(gain) : (R)0;
  }
  __syncthreads();
  const int half = Ms / 2;
  for (int kc = 0; kc < K; kc += KCH) {
    const int kn = min(KCH, K - kc);
    // g[i][k - kc]: Philox (j = s*half + t) -> g[2t], g[2t+1]; counter-based, so
    // users that do not see subarray s (amp 0, their rows are zero) are skipped
    for (int e = tid; e < half * kn; e += blockDim.x) {
      int kk = e / half, t = e % half, k = kc + kk;
      if (amp[k] == (R)0) continue;
      uint4 z = philox4x32_10(make_uint4((uint32_t)(s * half + t), (uint32_t)k | (PURPOSE_FADE << 24), b_lo, b_hi), k0, k1);
      double r0 = sqrt(-log(u01(z.x))), r1 = sqrt(-log(u01(z.z)));
      double s0, c0, s1, c1;  // theta = 2 pi u
      sincospi(2.0 * u01(z.y), &s0, &c0);
      sincospi(2.0 * u01(z.w), &s1, &c1);
      g[(2 * t) * KCH + kk] = mk<R>((R)(r0 * c0), (R)(r0 * s0));
      g[(2 * t + 1) * KCH + kk] = mk<R>((R)(r1 * c1), (R)(r1 * s1));
    }
    __syncthreads();
    for (int e = tid; e < Ms * kn; e += blockDim.x) {
      int i = e / kn, kk = e % kn, k = kc + kk;
      R a = amp[k];
      C acc = mk<R>(0, 0);
      if (a != (R)0) {
        for (int j = 0; j < Ms; ++j) {
          R rij = rs[i * Ms + j];
          C gj = g[j * KCH + kk];
          acc.x += rij * gj.x;
          acc.y += rij * gj.y;
        }
        acc.x *= a; acc.y *= a;
      }
      H[(bl * M + (int64_t)s * Ms + i) * K + k] = acc;
    }
    __syncthreads();
  }
}

// Box-Muller pair from two Philox words: complex64 in fp32 (logf / sincospif,
// ~1e-7 relative: far inside the c64 parity bound), complex128 in fp64 (the
// oracle's arithmetic).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& re, float& im) {
  const float u = __fmaf_rn((float)a, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float v = __fmaf_rn((float)b, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrtf(-logf(u));
  float sn, cs;
  sincospif(2.0f * v, &sn, &cs);
  re = r * cs;
  im = r * sn;
}
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, double& re, double& im) {
  const double r = sqrt(-log(u01(a)));
  double sn, cs;
  sincospi(2.0 * u01(b), &sn, &cs);
  re = r * cs;
  im = r * sn;
}

// One CTA per realization (S * K <= VIS_BITS): the users' gains and visibility
// masks are drawn once per realization (not once per subarray), then the CTA
// walks the subarrays; fading is drawn only for the visible (user, subarray)
// pairs (counter-based stream: the same values as chan_kernel / the oracle).
constexpr int VIS_BITS = 1 << 14;
template <typename R>
__global__ void __launch_bounds__(256, 3)
chan_real_kernel(uint64_t seed, int64_t first, int S, int Ms, int K, double p,
                 const double* __restrict__ Rsqrt, double beta_bar, double dmin, double dmax,
                 cplx<R>* __restrict__ H, int32_t* __restrict__ status) {
  using C = cplx<R>;
  const int64_t bl = blockIdx.x;
  const uint64_t bg = (uint64_t)(first + bl);
  const uint32_t b_lo = (uint32_t)bg, b_hi = (uint32_t)(bg >> 32);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int M = S * Ms;
  extern __shared__ double smem[];
  R* rs = (R*)smem;                        // Ms x Ms
  R* amp = rs + Ms * Ms;                   // K
  uint32_t* vis = (uint32_t*)(amp + ((K + 1) & ~1));  // [K][ceil(S/32)] visibility bits
  const int sw = (S + 31) / 32;
  C* g = (C*)(vis + ((K * sw + 3) & ~3));  // Ms x KCH (16-B aligned for double2)
  const int tid = threadIdx.x;
  for (int e = tid; e < Ms * Ms; e += blockDim.x) rs[(e % Ms) * Ms + e / Ms] = (R)Rsqrt[e];  // transposed
  const int nq = (S + 3) / 4;
  for (int k = tid; k < K; k += blockDim.x) {
    uint4 x = philox4x32_10(make_uint4(0u, (uint32_t)k | (PURPOSE_DIST << 24), b_lo, b_hi), k0, k1);
    double d = dmin + (dmax - dmin) * u01(x.x);
    double bdb = -35.3 - 37.6 * log10(d);
    double gain = pow(10.0, bdb / 10.0) / beta_bar;
    bool found = false;
    for (int att = 0; att < MAX_VIS_ATTEMPTS && !found; ++att) {
      for (int w = 0; w < sw; ++w) vis[k * sw + w] = 0u;
      for (int q = 0; q < nq; ++q) {
        uint4 y = philox4x32_10(make_uint4((uint32_t)(att * nq + q), (uint32_t)k | (PURPOSE_VIS << 24), b_lo, b_hi), k0, k1);
        uint32_t wv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int ss = 4 * q + e;
          if (ss < S && u01(wv[e]) < p) {
            vis[k * sw + (ss >> 5)] |= 1u << (ss & 31);
            found = true;
          }
        }
      }
    }
    if (!found) status[bl] = XL_STATUS_NO_VISIBLE;
    amp[k] = found ? (R)sqrt(gain) : (R)0;
  }
  __syncthreads();
  // per subarray: compact the users that see it, draw their fading, then
  // y = R^{1/2} g as a register-tiled (Ms x Ms) x (Ms x users) product
  // (thread = one user x 8 rows; the R^{1/2} column is a warp broadcast)
  const int half = Ms / 2;
  int* vlist = (int*)(g + (size_t)Ms * KCH);  // K compacted user indices
  __shared__ int nvis;
  for (int s = 0; s < S; ++s) {
    if (tid < 32) {  // warp 0: ballot compaction in user order
      int n = 0;
      for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + tid;
        const bool v = k < K && ((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, v);
        if (v) vlist[n + __popc(bal & ((1u << tid) - 1u))] = k;
        n += __popc(bal);
      }
      if (tid == 0) nvis = n;
    }
    // zero rows of the users that do not see subarray s (coalesced, masked)
    if (blockDim.x % K == 0) {  // a fixed user per thread
      const int k = tid % K;
      if (!((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u)) {
        C* hp = H + (bl * M + (int64_t)s * Ms) * K + k;
        for (int i = tid / K; i < Ms; i += blockDim.x / K) hp[(int64_t)i * K] = mk<R>(0, 0);
      }
    } else {
      for (int e = tid; e < Ms * K; e += blockDim.x) {
        const int i = e / K, k = e % K;
        if (!((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u)) H[(bl * M + (int64_t)s * Ms + i) * K + k] = mk<R>(0, 0);
      }
    }
    __syncthreads();
    const int nv = nvis;
    for (int vc = 0; vc < nv; vc += KCH) {
      const int kn = min(KCH, nv - vc);
      for (int e = tid; e < half * kn; e += blockDim.x) {
        const int kk = e / half, t = e % half, k = vlist[vc + kk];
        uint4 z = philox4x32_10(make_uint4((uint32_t)(s * half + t), (uint32_t)k | (PURPOSE_FADE << 24), b_lo, b_hi), k0, k1);
        R r0, i0, r1, i1;
        box_muller(z.x, z.y, r0, i0);
        box_muller(z.z, z.w, r1, i1);
        g[(2 * t) * KCH + kk] = mk<R>(r0, i0);
        g[(2 * t + 1) * KCH + kk] = mk<R>(r1, i1);
      }
      __syncthreads();
      constexpr int TR = 8;  // rows per thread
      for (int w = tid; w < KCH * (Ms / TR); w += blockDim.x) {
        const int kk = w % KCH, i0 = TR * (w / KCH);
        if (kk >= kn) continue;
        R ar[TR], ai[TR];
#pragma unroll
        for (int u = 0; u < TR; ++u) ar[u] = ai[u] = (R)0;
#pragma unroll 4
        for (int j = 0; j < Ms; ++j) {
          const C gj = g[j * KCH + kk];
          const R* col = rs + j * Ms + i0;  // R^{1/2} stored transposed: col[u] = R^{1/2}[i0 + u][j]
#pragma unroll
          for (int u = 0; u < TR; ++u) {
            ar[u] += col[u] * gj.x;
            ai[u] += col[u] * gj.y;
          }
        }
        const int k = vlist[vc + kk];
        const R a = amp[k];
        C* hp = H + (bl * M + (int64_t)s * Ms + i0) * K + k;
#pragma unroll
        for (int u = 0; u < TR; ++u) hp[(int64_t)u * K] = mk<R>(ar[u] * a, ai[u] * a);
      }
      __syncthreads();
    }
  }
}

// complex64, Ms = 64: chan_real_kernel with y = R^{1/2} g on the tensor cores
// (mma.sync m16n8k8 TF32, 3xTF32: R^{1/2} = Rh + Rl, g = gh + gl, y = Rh gh +
// Rh gl + Rl gh with fp32 accumulation, ~1e-7 relative -- the SIMT FFMA loop
// was 55% of the kernel's instructions).  Per subarray and chunk of <= 64
// visible users the (64 x 64) x (64 x 2 users) real product is 4 x 16 output
// tiles of 16 x 8 over the 8 warps (two column tiles each, all four row tiles).
__device__ __forceinline__ uint32_t tf32_of(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
constexpr int TC_MS = 64, TC_RS = TC_MS + 4, TC_GS = 2 * KCH + 4;  // padded row strides (floats)

__global__ void __launch_bounds__(256, 2)
chan_tc_kernel(uint64_t seed, int64_t first, int S, int K, double p, const double* __restrict__ Rsqrt,
               double beta_bar, double dmin, double dmax, float2* __restrict__ H, int32_t* __restrict__ status) {
  constexpr int Ms = TC_MS;
  const int64_t bl = blockIdx.x;
  const uint64_t bg = (uint64_t)(first + bl);
  const uint32_t b_lo = (uint32_t)bg, b_hi = (uint32_t)(bg >> 32);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int M = S * Ms;
  extern __shared__ double smem[];
  uint32_t* rsh = (uint32_t*)smem;                 // [Ms][TC_RS] tf32 hi of R^{1/2}
  uint32_t* rsl = rsh + Ms * TC_RS;                // lo
  float* gf = (float*)(rsl + Ms * TC_RS);          // [Ms][TC_GS]: (Re, Im) of the chunk's users
  float* amp = gf + Ms * TC_GS;                    // K
  uint32_t* vis = (uint32_t*)(amp + ((K + 3) & ~3));
  const int sw = (S + 31) / 32;
  int* vlist = (int*)(vis + ((K * sw + 3) & ~3));  // K compacted user indices
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < Ms * Ms; e += blockDim.x) {
    const float x = (float)Rsqrt[e];
    const uint32_t h = tf32_of(x);
    rsh[(e / Ms) * TC_RS + e % Ms] = h;
    rsl[(e / Ms) * TC_RS + e % Ms] = tf32_of(x - __uint_as_float(h));
  }
  const int nq = (S + 3) / 4;
  for (int k = tid; k < K; k += blockDim.x) {
    uint4 x = philox4x32_10(make_uint4(0u, (uint32_t)k | (PURPOSE_DIST << 24), b_lo, b_hi), k0, k1);
    double d = dmin + (dmax - dmin) * u01(x.x);
    double bdb = -35.3 - 37.6 * log10(d);
    double gain = pow(10.0, bdb / 10.0) / beta_bar;
    bool found = false;
    for (int att = 0; att < MAX_VIS_ATTEMPTS && !found; ++att) {
      for (int w = 0; w < sw; ++w) vis[k * sw + w] = 0u;
      for (int q = 0; q < nq; ++q) {
        uint4 y = philox4x32_10(make_uint4((uint32_t)(att * nq + q), (uint32_t)k | (PURPOSE_VIS << 24), b_lo, b_hi), k0, k1);
        uint32_t wv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int ss = 4 * q + e;
          if (ss < S && u01(wv[e]) < p) {
            vis[k * sw + (ss >> 5)] |= 1u << (ss & 31);
            found = true;
          }
        }
      }
    }
    if (!found) status[bl] = XL_STATUS_NO_VISIBLE;
    amp[k] = found ? (float)sqrt(gain) : 0.0f;
  }
  __syncthreads();
  const int half = Ms / 2;
  __shared__ int nvis;
  const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  for (int s = 0; s < S; ++s) {
    if (tid < 32) {  // warp 0: ballot compaction in user order
      int n = 0;
      for (int kb = 0; kb < K; kb += 32) {
        const int k = kb + tid;
        const bool v = k < K && ((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, v);
        if (v) vlist[n + __popc(bal & ((1u << tid) - 1u))] = k;
        n += __popc(bal);
      }
      if (tid == 0) nvis = n;
    }
    // zero rows of the users that do not see subarray s
    if (blockDim.x % K == 0) {
      const int k = tid % K;
      if (!((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u)) {
        float2* hp = H + (bl * M + (int64_t)s * Ms) * K + k;
        for (int i = tid / K; i < Ms; i += blockDim.x / K) hp[(int64_t)i * K] = make_float2(0.0f, 0.0f);
      }
    } else {
      for (int e = tid; e < Ms * K; e += blockDim.x) {
        const int i = e / K, k = e % K;
        if (!((vis[k * sw + (s >> 5)] >> (s & 31)) & 1u)) H[(bl * M + (int64_t)s * Ms + i) * K + k] = make_float2(0.0f, 0.0f);
      }
    }
    __syncthreads();
    const int nv = nvis;
    for (int vc = 0; vc < nv; vc += KCH) {
      const int kn = min(KCH, nv - vc);
      for (int e = tid; e < half * kn; e += blockDim.x) {
        const int kk = e / half, t = e % half, k = vlist[vc + kk];
        uint4 z = philox4x32_10(make_uint4((uint32_t)(s * half + t), (uint32_t)k | (PURPOSE_FADE << 24), b_lo, b_hi), k0, k1);
        float r0, i0, r1, i1;
        box_muller(z.x, z.y, r0, i0);
        box_muller(z.z, z.w, r1, i1);
        *reinterpret_cast<float2*>(gf + (2 * t) * TC_GS + 2 * kk) = make_float2(r0, i0);
        *reinterpret_cast<float2*>(gf + (2 * t + 1) * TC_GS + 2 * kk) = make_float2(r1, i1);
      }
      __syncthreads();
      // warp w: column tiles 2w, 2w + 1 (columns 16 w .. 16 w + 15 = users 8 w .. 8 w + 7)
      const int ncol = 2 * kn;
      if (16 * warp < ncol) {
        float acc[4][2][4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0f;
#pragma unroll 2
        for (int kk0 = 0; kk0 < Ms; kk0 += 8) {
          uint32_t bh[2][2], blo[2][2];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int col = 16 * warp + 8 * nt + gq;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const float x = gf[(kk0 + tq + 4 * h2) * TC_GS + col];
              const uint32_t hx = tf32_of(x);
              bh[nt][h2] = hx;
              blo[nt][h2] = tf32_of(x - __uint_as_float(hx));
            }
          }
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int r0 = 16 * mt + gq;
            const uint32_t ah[4] = {rsh[r0 * TC_RS + kk0 + tq], rsh[(r0 + 8) * TC_RS + kk0 + tq],
                                    rsh[r0 * TC_RS + kk0 + tq + 4], rsh[(r0 + 8) * TC_RS + kk0 + tq + 4]};
            const uint32_t al[4] = {rsl[r0 * TC_RS + kk0 + tq], rsl[(r0 + 8) * TC_RS + kk0 + tq],
                                    rsl[r0 * TC_RS + kk0 + tq + 4], rsl[(r0 + 8) * TC_RS + kk0 + tq + 4]};
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma_tf32(acc[mt][nt], ah, bh[nt][0], bh[nt][1]);
              mma_tf32(acc[mt][nt], ah, blo[nt][0], blo[nt][1]);
              mma_tf32(acc[mt][nt], al, bh[nt][0], bh[nt][1]);
            }
          }
        }
        // c0, c1: row 16 mt + gq, columns 2 tq, 2 tq + 1 of the tile = (Re, Im) of one user
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int kk = 8 * warp + 4 * nt + tq;
          if (kk < kn) {
            const int k = vlist[vc + kk];
            const float a = amp[k];
            float2* hp = H + (bl * M + (int64_t)s * Ms) * K + k;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
              hp[(int64_t)(16 * mt + gq) * K] = make_float2(acc[mt][nt][0] * a, acc[mt][nt][1] * a);
              hp[(int64_t)(16 * mt + gq + 8) * K] = make_float2(acc[mt][nt][2] * a, acc[mt][nt][3] * a);
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

int launch_channel(int dtype, uint64_t seed, int64_t first, int64_t B, int S, int Ms,
                   int K, double p, const double* Rsqrt, double beta_bar, double dmin,
                   double dmax, void* H, int32_t* status, cudaStream_t st) {
  if (S > 65535 || (Ms & 1)) { set_error("channel: unsupported S/Ms"); return XL_ERR_UNSUPPORTED; }
  size_t rsz = dtype == XL_C64 ? 4 : 8;
  if (dtype == XL_C64 && Ms == TC_MS && (int64_t)S * K <= VIS_BITS && B <= 0x7fffffff) {
    // complex64, Ms = 64: R^{1/2} g on the tensor cores (3xTF32)
    const int sw = (S + 31) / 32;
    const size_t smem = 4 * (2 * (size_t)TC_MS * TC_RS + (size_t)TC_MS * TC_GS + ((K + 3) & ~3) +
                             (size_t)((K * sw + 3) & ~3) + (size_t)K);
    cudaFuncSetAttribute(chan_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chan_tc_kernel<<<(unsigned)B, 256, smem, st>>>(seed, first, S, K, p, Rsqrt, beta_bar, dmin, dmax, (float2*)H,
                                                   status);
    return check_launch("channel_generate");
  }
  if ((int64_t)S * K <= VIS_BITS && Ms % 8 == 0 && B <= 0x7fffffff) {  // one CTA per realization
    const int sw = (S + 31) / 32;
    size_t smem = rsz * ((size_t)Ms * Ms + ((K + 1) & ~1)) + 4 * (size_t)((K * sw + 3) & ~3) +
                  2 * rsz * (size_t)Ms * KCH + 4 * (size_t)K;
    if (dtype == XL_C64) {
      cudaFuncSetAttribute(chan_real_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      chan_real_kernel<float><<<(unsigned)B, 256, smem, st>>>(seed, first, S, Ms, K, p, Rsqrt, beta_bar, dmin, dmax,
                                                              (float2*)H, status);
    } else {
      cudaFuncSetAttribute(chan_real_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      chan_real_kernel<double><<<(unsigned)B, 256, smem, st>>>(seed, first, S, Ms, K, p, Rsqrt, beta_bar, dmin, dmax,
                                                               (double2*)H, status);
    }
    return check_launch("channel_generate");
  }
  dim3 grid((unsigned)B, (unsigned)S);
  size_t smem = rsz * ((size_t)Ms * Ms + ((K + 1) & ~1)) + 2 * rsz * (size_t)Ms * KCH;
  if (dtype == XL_C64) {
    cudaFuncSetAttribute(chan_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chan_kernel<float><<<grid, 256, smem, st>>>(seed, first, S, Ms, K, p, Rsqrt, beta_bar, dmin, dmax, (float2*)H, status);
  } else {
    cudaFuncSetAttribute(chan_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chan_kernel<double><<<grid, 256, smem, st>>>(seed, first, S, Ms, K, p, Rsqrt, beta_bar, dmin, dmax, (double2*)H, status);
  }
  return check_launch("channel_generate");
}

}  // namespace xl
