// Microbenchmark: per-SM cp.async.bulk streaming with an NS x SB smem ring and
// no compute -> achievable DRAM read bandwidth vs bytes in flight per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(128, 1) stream(const char* src, size_t per_cta, int SB, int NS, unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* ring = smem + 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char* base = src + blockIdx.x * per_cta;
  size_t n = per_cta / SB;
  unsigned long long acc = 0;
  for (size_t i = 0; i < n + NS; ++i) {
    if (i >= (size_t)NS) {  // consume item i - NS
      size_t j = i - NS; int s = j % NS; uint32_t par = (j / NS) & 1, done = 0;
      do { asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(done) : "r"(su32(&bars[s])), "r"(par) : "memory"); } while (!done);
      acc += *(volatile int*)(ring + s * SB);
    }
    if (i < n) {
      int s = i % NS;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(SB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + s * SB)), "l"(base + i * SB), "r"(SB), "r"(su32(&bars[s])) : "memory");
    }
  }
  sink[blockIdx.x] = acc;
}
int main() {
  int nsm = 148; size_t per_cta = 64ull << 20;  // 64 MB per CTA -> 9.5 GB total
  char* src; cudaMalloc(&src, per_cta * nsm); cudaMemset(src, 1, per_cta * nsm);
  unsigned long long* sink; cudaMalloc(&sink, nsm * 8);
  int cfgs[][2] = {{32768, 3}, {16384, 6}, {32768, 6}, {65536, 3}, {16384, 12}, {8192, 12}};
  for (auto& c : cfgs) {
    int SB = c[0], NS = c[1]; size_t smem = 1024 + (size_t)SB * NS;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    stream<<<nsm, 128, smem>>>(src, per_cta, SB, NS, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) stream<<<nsm, 128, smem>>>(src, per_cta, SB, NS, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("SB=%6d NS=%2d in-flight=%4d KB/SM: %.0f GB/s  (%s)\n", SB, NS, SB * NS / 1024,
           3.0 * per_cta * nsm / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
