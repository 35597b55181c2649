// Microbenchmark: per-SM cost of writing one 32 KB W^T tile (64 antennas x
// 128 components fp32, row-major in HBM) from 4 warps, as the fused kernel's
// epilogue does.  mode 0: 64 x st.global.cs.f32 per thread (128 B/warp-instr);
// mode 1: 16 x st.global.cs.v4.f32 per thread (4-lane transposed data);
// mode 2: 64 x st.shared.f32 into a staging tile + one cp.async.bulk store.
// Reports cycles per tile (clock64 around the loop, all 148 SMs active).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(128, 1) k(float* dst, int iters, int mode, long long* cyc) {
  extern __shared__ __align__(1024) char smem[];
  float* stg = reinterpret_cast<float*>(smem);
  const int r = threadIdx.x;  // component 0..127
  float d[64];
#pragma unroll
  for (int a = 0; a < 64; ++a) d[a] = r * 0.5f + a;
  float* base = dst + (size_t)blockIdx.x * iters * 64 * 128;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float* w = base + (size_t)it * 64 * 128;
    if (mode == 0) {
#pragma unroll
      for (int a = 0; a < 64; ++a) __stcs(w + a * 128 + r, d[a] * 1.5f);
    } else if (mode == 1) {
      float4* w4 = reinterpret_cast<float4*>(w);
      const int g = r >> 2, i = r & 3;  // 32 column groups of 4 components
#pragma unroll
      for (int q = 0; q < 16; ++q)      // antenna a = 4 q + i
        __stcs(w4 + (4 * q + i) * 32 + g, make_float4(d[4 * q], d[4 * q + 1], d[4 * q + 2], d[4 * q + 3]));
    } else {
#pragma unroll
      for (int a = 0; a < 64; ++a) stg[a * 128 + r] = d[a] * 1.5f;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (r == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(w), "r"(su32(stg)), "r"(32768) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
    }
  }
  if (mode == 2 && r == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (r == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  const int nsm = 148, iters = 256;
  float* dst; cudaMalloc(&dst, (size_t)nsm * iters * 32768);
  long long* cyc; cudaMallocManaged(&cyc, nsm * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid : {1, nsm}) {
      k<<<grid, 128, 32768>>>(dst, iters, mode, cyc);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<grid, 128, 32768>>>(dst, iters, mode, cyc);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double mean = 0; for (int i = 0; i < grid; ++i) mean += cyc[i]; mean /= grid;
      printf("mode %d grid %3d: %.0f cycles per 32 KB tile, %.0f GB/s total (%s)\n", mode, grid, mean / iters,
             (double)grid * iters * 32768 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
