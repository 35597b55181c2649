// Microbenchmark: achievable HBM throughput for the fused kernel's traffic
// mix (per SM: bulk TMA reads into a 3 x 32 KB ring, writes at half the read
// volume) with different store flavours.
//   mode 0: reads only   1: + st.global.cs.f32 (128 B/warp/instr)
//   2: + st.global.cs.v4.f32   3: + cp.async.bulk smem->global stores
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do { asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory"); } while (!done);
}
__global__ void __launch_bounds__(160, 1) k(const char* src, float* dst, size_t per_cta, int mode) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = (uint64_t*)smem;       // [3]
  uint64_t* empty = full + 3;             // [3]
  char* ring = smem + 1024;
  const int NS = 3, SB = 32768;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  float* wbase = dst + blockIdx.x * (per_cta / 2) / 4;
  const size_t n = per_cta / SB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) {
    if (lane == 0)
      for (size_t i = 0; i < n; ++i) {
        int s = i % NS;
        if (i >= NS) wait(&empty[s], ((i / NS) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + s * SB)), "l"(base + i * SB), "r"(SB), "r"(su32(&full[s])) : "memory");
      }
    return;
  }
  // warps 0-3: consume; on odd items write 32 KB (= half the read volume)
  for (size_t i = 0; i < n; ++i) {
    int s = i % NS;
    wait(&full[s], (i / NS) & 1);
    float acc = *(volatile float*)(ring + s * SB + 4 * threadIdx.x);
    if (mode != 0 && (i & 1)) {
      float* w = wbase + (i / 2) * (SB / 4);
      if (mode == 1) {
        for (int a = 0; a < 64; ++a) __stcs(w + a * 128 + threadIdx.x, acc + a);
      } else if (mode == 2) {
        float4* w4 = reinterpret_cast<float4*>(w);
        for (int a = 0; a < 16; ++a) __stcs(w4 + a * 128 + threadIdx.x, make_float4(acc, acc, acc, a));
      } else {
        __syncwarp();
        asm volatile("bar.sync 1, 128;");
        if (threadIdx.x == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(w), "r"(su32(ring + s * SB)), "r"(SB) : "memory");
          asm volatile("cp.async.bulk.commit_group;");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        asm volatile("bar.sync 1, 128;");
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
  }
}
int main() {
  int nsm = 148; size_t per_cta = 48ull << 20;
  char* src; cudaMalloc(&src, per_cta * nsm); cudaMemset(src, 1, per_cta * nsm);
  float* dst; cudaMalloc(&dst, per_cta * nsm / 2);
  size_t smem = 1024 + 3 * 32768;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<nsm, 160, smem>>>(src, dst, per_cta, mode);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) k<<<nsm, 160, smem>>>(src, dst, per_cta, mode);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 3.0 * per_cta * nsm * (mode ? 1.5 : 1.0);
    printf("mode %d: %.0f GB/s total (%s)\n", mode, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
