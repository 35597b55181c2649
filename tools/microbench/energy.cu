// Energy per byte of the data paths the fused kernel uses: TMA bulk reads from
// HBM vs from L2, coalesced 4-B/lane streaming stores, and both mixed.  Each
// config loops ~3 s; power comes from nvidia-smi sampled alongside (see
// tools/microbench/energy.sh), matched by the printed wall-clock windows.
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// mode 0: TMA read ring over a per-CTA window of `win` bytes repeated to `per_cta`
// mode 1: coalesced st.global.cs 4 B/lane over per_cta bytes (512 threads)
// mode 2: both (reads by thread 0's TMA ring, stores by warps 1..15)
__global__ void __launch_bounds__(512, 1) kern(char* src, char* dst, size_t per_cta, size_t win, int mode,
                                               unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  const int SB = 32768, NS = 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* ring = smem + 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (mode != 1 && threadIdx.x == 0) {
    const char* base = src + blockIdx.x * win;
    size_t n = per_cta / SB, nw = win / SB;
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
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + s * SB)), "l"(base + (i % nw) * SB), "r"(SB), "r"(su32(&bars[s])) : "memory");
      }
    }
    sink[blockIdx.x] = acc;
  }
  if ((mode == 1 || mode == 2) && threadIdx.x >= 32) {
    const int t = threadIdx.x - 32, nt = 480;
    float* d = reinterpret_cast<float*>(dst + blockIdx.x * win);
    const size_t nw = win / 4;
    for (size_t r = 0; r < per_cta / win; ++r)
      for (size_t i = t; i < nw; i += nt) __stcs(d + i, (float)(i + r));
  }
  if (mode == 3 && threadIdx.x >= 32) {  // 16 B per lane, default policy
    const int t = threadIdx.x - 32, nt = 480;
    float4* d = reinterpret_cast<float4*>(dst + blockIdx.x * win);
    const size_t nw = win / 16;
    for (size_t r = 0; r < per_cta / win; ++r)
      for (size_t i = t; i < nw; i += nt) d[i] = make_float4((float)(i + r), 1.f, 2.f, 3.f);
  }
  if (mode == 4 && threadIdx.x >= 32) {  // 4 B per lane, default policy
    const int t = threadIdx.x - 32, nt = 480;
    float* d = reinterpret_cast<float*>(dst + blockIdx.x * win);
    const size_t nw = win / 4;
    for (size_t r = 0; r < per_cta / win; ++r)
      for (size_t i = t; i < nw; i += nt) d[i] = (float)(i + r);
  }
  if (mode == 6 && threadIdx.x >= 32) {  // 16 B per lane, streaming (.cs)
    const int t = threadIdx.x - 32, nt = 480;
    float4* d = reinterpret_cast<float4*>(dst + blockIdx.x * win);
    const size_t nw = win / 16;
    for (size_t r = 0; r < per_cta / win; ++r)
      for (size_t i = t; i < nw; i += nt) __stcs(d + i, make_float4((float)(i + r), 1.f, 2.f, 3.f));
  }
  if (mode == 8 && threadIdx.x >= 32) {  // 8 B per lane, streaming (.cs)
    const int t = threadIdx.x - 32, nt = 480;
    float2* d = reinterpret_cast<float2*>(dst + blockIdx.x * win);
    const size_t nw = win / 8;
    for (size_t r = 0; r < per_cta / win; ++r)
      for (size_t i = t; i < nw; i += nt) __stcs(d + i, make_float2((float)(i + r), 1.f));
  }
  if (mode == 7 && threadIdx.x == 0) {  // TMA bulk stores with an L2 evict_first hint
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    char* d = dst + blockIdx.x * win;
    size_t n = per_cta / SB, nw = win / SB;
    for (size_t i = 0; i < n; ++i) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(d + (i % nw) * SB), "r"(su32(ring + (i % NS) * SB)), "r"(SB), "l"(pol) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (mode == 5 && threadIdx.x == 0) {  // TMA bulk stores of 32 KiB smem chunks, 4 in flight
    char* d = dst + blockIdx.x * win;
    size_t n = per_cta / SB, nw = win / SB;
    for (size_t i = 0; i < n; ++i) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + (i % nw) * SB), "r"(su32(ring + (i % NS) * SB)), "r"(SB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main(int argc, char** argv) {
  const int nsm = 148;
  const size_t per_cta = 64ull << 20;  // bytes per CTA per launch
  char *src, *dst;
  cudaMalloc(&src, per_cta * nsm);
  cudaMalloc(&dst, per_cta * nsm);
  cudaMemset(src, 1, per_cta * nsm);
  unsigned long long* sink;
  cudaMalloc(&sink, nsm * 8);
  const size_t smem = 1024 + 4 * 32768;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct C { const char* name; int mode; size_t win; } cfgs[] = {
      {"idle", -1, 0}, {"read_hbm", 0, per_cta}, {"read_l2_256K", 0, 256 << 10}, {"store_hbm", 1, per_cta},
      {"read_hbm+store", 2, per_cta}, {"read_l2+store", 2, 256 << 10},
      {"store_l2_256K", 1, 256 << 10}, {"store128_hbm", 3, per_cta}, {"store128_l2", 3, 256 << 10},
      {"store_wb_hbm", 4, per_cta}, {"tma_store_hbm", 5, per_cta}, {"tma_store_l2", 5, 256 << 10},
      {"store128cs_hbm", 6, per_cta}, {"store64cs_hbm", 8, per_cta}, {"tma_store_ef_hbm", 7, per_cta}};
  for (auto& c : cfgs) {
    auto t0 = std::chrono::system_clock::now();
    double secs = 0, bytes = 0;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    if (c.mode < 0) {
      while (std::chrono::duration<double>(std::chrono::system_clock::now() - t0).count() < 3.0) {}
    } else {
      float tot = 0;
      int launches = 0;
      while (std::chrono::duration<double>(std::chrono::system_clock::now() - t0).count() < 3.0) {
        cudaEventRecord(a);
        kern<<<nsm, 512, smem>>>(src, dst, per_cta, c.win, c.mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        tot += ms; ++launches;
      }
      secs = tot * 1e-3;
      bytes = (double)per_cta * nsm * launches * (c.mode == 2 ? 2 : 1);
    }
    auto t1 = std::chrono::system_clock::now();
    printf("%-16s t0 %.3f t1 %.3f  %.0f GB/s (%s)\n", c.name,
           std::chrono::duration<double>(t0.time_since_epoch()).count(),
           std::chrono::duration<double>(t1.time_since_epoch()).count(), secs > 0 ? bytes / secs / 1e9 : 0.0,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
}
