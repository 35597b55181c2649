// Shared device helpers for the xlmimo B200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xlmimo_b200.h"

namespace xl {

template <typename R> struct ctype;
template <> struct ctype<float> { using T = float2; };
template <> struct ctype<double> { using T = double2; };
template <typename R> using cplx = typename ctype<R>::T;

template <typename R> __host__ __device__ __forceinline__ cplx<R> mk(R re, R im) {
  cplx<R> z; z.x = re; z.y = im; return z;
}
template <typename C> __host__ __device__ __forceinline__ C cadd(C a, C b) { a.x += b.x; a.y += b.y; return a; }
template <typename C> __host__ __device__ __forceinline__ C csub(C a, C b) { a.x -= b.x; a.y -= b.y; return a; }
template <typename C> __host__ __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }
template <typename C, typename R> __host__ __device__ __forceinline__ C cscale(C a, R s) { a.x *= s; a.y *= s; return a; }
// acc += a * b
template <typename C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename C> __device__ __forceinline__ void cfma_conj(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}
template <typename C> __device__ __forceinline__ auto cabs2(C a) { return a.x * a.x + a.y * a.y; }

__device__ __forceinline__ float  warp_sum(float v)  { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }
__device__ __forceinline__ double warp_sum(double v) { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }

// Host-side error slot (xl_abi.cu).
void set_error(const char* fmt, ...);
int check_launch(const char* what);

}  // namespace xl
