// Microbenchmark: does an L2 evict_last policy on cp.async.bulk loads keep a
// working set resident while other data streams through with evict_first?
// phase 1: load X (keep policy), phase 2: stream Y (evict_first), phase 3:
// reload X.  Compare dram__bytes_read under ncu for the policy variants.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void load(const char* src, size_t bytes, char* buf, uint64_t* bar, uint32_t& ph, uint64_t pol) {
  for (size_t off = 0; off < bytes; off += 32768) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32768) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(su32(buf)), "l"(src + off), "r"(32768), "r"(su32(bar)), "l"(pol) : "memory");
    uint32_t done = 0;
    do { asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(done) : "r"(su32(bar)), "r"(ph) : "memory"); } while (!done);
    ph ^= 1;
  }
}
__global__ void k(const char* X, size_t xs, const char* Y, size_t ys, int mode) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* bar = (uint64_t*)smem;
  if (mode >= 3) {  // mode 3: X load (evict_last) then all threads write Y with st.global.cs; 4: same, no X reload gap
    const size_t xper = xs / gridDim.x, yper = ys / gridDim.x;
    uint64_t last;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t ph = 0;
    if (threadIdx.x == 0) load(X + blockIdx.x * xper, xper, smem + 1024, bar, ph, last);
    __syncthreads();
    float4* yw = (float4*)(const_cast<char*>(Y) + blockIdx.x * yper);
    for (size_t i = threadIdx.x; i < yper / 16; i += blockDim.x) __stcs(yw + i, make_float4(1.f, 2.f, 3.f, 4.f));
    __syncthreads();
    if (threadIdx.x == 0) load(X + blockIdx.x * xper, xper, smem + 1024, bar, ph, last);
    return;
  }
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint64_t first, last, normal;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(normal));
  uint32_t ph = 0;
  const size_t xper = xs / gridDim.x, yper = ys / gridDim.x;
  load(X + blockIdx.x * xper, xper, smem + 1024, bar, ph, mode == 0 ? last : normal);
  if (mode == 0 || mode == 1) load(Y + blockIdx.x * yper, yper, smem + 1024, bar, ph, first);
  load(X + blockIdx.x * xper, xper, smem + 1024, bar, ph, first);
}
int main(int argc, char** argv) {
  size_t xs = (size_t)atoi(argv[1]) << 20, ys = (size_t)atoi(argv[2]) << 20;
  int mode = atoi(argv[3]);  // 0 evict_last, 1 evict_normal, 2 no Y stream
  xs = xs / (148 * 32768) * 148 * 32768; ys = ys / (148 * 32768) * 148 * 32768;
  char *X, *Y; cudaMalloc(&X, xs); cudaMalloc(&Y, ys); cudaMemset(X, 1, xs); cudaMemset(Y, 2, ys);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 32768);
  const int nt = mode >= 3 ? 256 : 32;
  k<<<148, nt, 1024 + 32768>>>(X, xs, Y, ys, mode);
  cudaDeviceSynchronize();
  k<<<148, nt, 1024 + 32768>>>(X, xs, Y, ys, mode);
  printf("X %zu MB Y %zu MB mode %d: %s\n", xs >> 20, ys >> 20, mode, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
