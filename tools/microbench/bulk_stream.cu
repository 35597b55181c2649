// Streaming rate of 1-D bulk copies (cp.async.bulk) from an L2-resident buffer
// into a shared-memory ring: one CTA per SM, NS stages of S bytes, each stage
// refilled as soon as it lands (no consumer work).  Reports bytes / SM cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bulk_stream bulk_stream.cu
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

namespace t {
#include "../../paper_2305_13925_b200/csrc/tc_ptx.cuh"
}
using namespace t;

__global__ void __launch_bounds__(32, 1) stream(const uint8_t* src, size_t span, int S, int NS, int total, int per_cta,
                                                long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (per_cta ? (size_t)blockIdx.x * span : 0);
  const uint64_t pol = policy_evict_normal();
  const long long t0 = clock64();
  for (int g = 0; g < total + NS; ++g) {
    if (g >= NS) mbar_wait(&full[(g - NS) % NS], ((g - NS) / NS) & 1);  // stage landed
    if (g < total) {
      const int s = g % NS;
      mbar_expect_tx(&full[s], S);
      bulk_g2s(sm + s * S, base + ((size_t)g * S) % span, S, &full[s], pol);
    }
  }
  out[blockIdx.x] = clock64() - t0;
}

// each stage filled by 8 lanes issuing S / 8 bytes each
__global__ void __launch_bounds__(32, 1) stream_mt(const uint8_t* src, size_t span, int S, int NS, int total,
                                                   long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * span;
  const uint64_t pol = policy_evict_normal();
  const int l = threadIdx.x;
  const long long t0 = clock64();
  for (int g = 0; g < total + NS; ++g) {
    if (g >= NS) mbar_wait(&full[(g - NS) % NS], ((g - NS) / NS) & 1);
    if (g < total) {
      const int s = g % NS;
      if (l == 0) mbar_expect_tx(&full[s], S);
      __syncwarp();
      if (l < 8) bulk_g2s(sm + s * S + l * (S / 8), base + ((size_t)g * S) % span + l * (S / 8), S / 8, &full[s], pol);
      __syncwarp();
    }
  }
  if (l == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t* buf;
  const size_t span = 512 * 1024;
  cudaMalloc(&buf, span * 148);
  cudaMemset(buf, 1, span * 148);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int per : {1})
    for (int S : {16384, 32768, 65536, 98304})
      for (int NS : {1, 2}) {
        if (S * NS > 200 * 1024) continue;
        const int total = (int)(4 * span / S);
        for (int grid : {1, 148}) {
          stream<<<grid, 32, S * NS>>>(buf, span, S, NS, total, per, d);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[148];
          cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
          double mx = 0;
          for (int i = 0; i < grid; ++i) mx = fmax(mx, (double)h[i]);
          printf("%s src, grid %3d, stage %6d B x %2d: %6.1f B/cycle/SM  %s\n", per ? "per-CTA" : "shared ", grid, S, NS,
                 (double)total * S / mx, cudaGetErrorString(e));
        }
      }
  // the same ring filled in 4 KiB pieces from 8 threads of the warp at once
  for (int S : {32768, 65536})
    for (int grid : {1, 148}) {
      stream_mt<<<grid, 32, S * 2>>>(buf, span, S, 2, (int)(4 * span / S), d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = fmax(mx, (double)h[i]);
      printf("8-thread issue, grid %3d, stage %6d B x 2: %6.1f B/cycle/SM  %s\n", grid, S, (double)(4 * span) / mx,
             cudaGetErrorString(e));
    }
  return 0;
}
