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
// One CTA per (realization, subarray): every CTA re-derives the users'
// gains/visibility (a few Philox calls) so H rows are written coalesced
// (row m = s*Ms + i holds all K users contiguously) without a workspace.
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
    // g[i][k - kc]: Philox (j = s*half + t) -> g[2t], g[2t+1]
    for (int e = tid; e < half * kn; e += blockDim.x) {
      int kk = e / half, t = e % half, k = kc + kk;
      uint4 z = philox4x32_10(make_uint4((uint32_t)(s * half + t), (uint32_t)k | (PURPOSE_FADE << 24), b_lo, b_hi), k0, k1);
      double r0 = sqrt(-log(u01(z.x))), th0 = 2.0 * M_PI * u01(z.y);
      double r1 = sqrt(-log(u01(z.z))), th1 = 2.0 * M_PI * u01(z.w);
      g[(2 * t) * KCH + kk] = mk<R>((R)(r0 * cos(th0)), (R)(r0 * sin(th0)));
      g[(2 * t + 1) * KCH + kk] = mk<R>((R)(r1 * cos(th1)), (R)(r1 * sin(th1)));
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

int launch_channel(int dtype, uint64_t seed, int64_t first, int64_t B, int S, int Ms,
                   int K, double p, const double* Rsqrt, double beta_bar, double dmin,
                   double dmax, void* H, int32_t* status, cudaStream_t st) {
  if (S > 65535 || (Ms & 1)) { set_error("channel: unsupported S/Ms"); return XL_ERR_UNSUPPORTED; }
  dim3 grid((unsigned)B, (unsigned)S);
  size_t rsz = dtype == XL_C64 ? 4 : 8;
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
