// Single-SM (and full-chip) memory interface: TMA bulk reads (ring of NS x 32 KiB),
// st.global.cs 4 B/lane stores by 8 warps, and both at once -- bytes per SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(288, 1) kern(const char* src, char* dst, size_t bytes, int mode, int NS,
                                               unsigned long long* sink, long long* clk) {
  extern __shared__ __align__(1024) char smem[];
  const int SB = 32768;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* ring = smem + 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long long t0 = clock64();
  if ((mode & 1) && threadIdx.x == 0) {
    const char* base = src + blockIdx.x * bytes;
    size_t n = bytes / SB;
    unsigned long long acc = 0;
    for (size_t i = 0; i < n + NS; ++i) {
      if (i >= (size_t)NS) {
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
  if ((mode & 2) && threadIdx.x >= 32) {  // 8 warps: each warp stores 128 B per instruction
    const int t = threadIdx.x - 32;
    float* d = reinterpret_cast<float*>(dst + blockIdx.x * bytes);
    const size_t n = bytes / 4;
    for (size_t i = t; i < n; i += 256) __stcs(d + i, (float)i);
  }
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
}
int main() {
  const size_t bytes = 256ull << 20;  // per CTA
  int nsm_list[] = {1, 148};
  char *src, *dst;
  cudaMalloc(&src, bytes * 148);
  cudaMalloc(&dst, bytes * 148);
  cudaMemset(src, 1, bytes * 148);
  unsigned long long* sink; cudaMalloc(&sink, 148 * 8);
  long long* clk; cudaMalloc(&clk, 148 * 8);
  for (int NS : {3, 4}) {
    size_t smem = 1024 + (size_t)NS * 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nsm : nsm_list)
      for (int mode : {1, 2, 3}) {
        kern<<<nsm, 288, smem>>>(src, dst, bytes / 8, mode, NS, sink, clk);  // warm
        kern<<<nsm, 288, smem>>>(src, dst, bytes, mode, NS, sink, clk);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        double bpc = (double)bytes / c;
        printf("NS=%d ctas=%3d mode=%s  %.1f B/clk per direction per SM  (%s)\n", NS, nsm,
               mode == 1 ? "read " : mode == 2 ? "write" : "both ", bpc, cudaGetErrorString(cudaGetLastError()));
      }
  }
}
