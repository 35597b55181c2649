// tcgen05.mma issue rate vs shape / operand source / B layout (one CTA per SM,
// thread 0 issues R x G MMAs into one accumulator, clock64 around them).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

namespace t {
#include "../../paper_2305_13925_b200/csrc/tc_ptx.cuh"
}
using namespace t;

__global__ void __launch_bounds__(128, 1) bench(int N, int mode, int bkmaj, int reps, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = slot;
  if (mode == 3 && tid < 32) {  // whole warp runs the loop; each MMA elects one lane in PTX
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    const uint32_t id = idesc(128, N, 0, 1);
    const uint64_t ad = sdesc(a, 128, 256);
    const uint64_t bd = sdesc(b, N * 16, 128);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const uint32_t dst = tmem + 256 + (uint32_t)((g & 1) * 128);
        asm volatile(
            "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dst),
            "l"(ad), "l"(bd), "r"(id), "r"(1));
      }
    }
    if (tid == 0) {
      commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  } else if (tid == 0 && mode != 3) {
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    // A K-major (SBO 256 = 8-row group, LBO 128 = K group); B MN-major
    // (LBO = K group stride, SBO 128 = N octet) or K-major (LBO 128, SBO 256)
    const uint32_t id = idesc(128, N, 0, bkmaj ? 0 : 1);
    const uint64_t ad = sdesc(a, 128, 256);
    const uint64_t bd = bkmaj ? sdesc(b, 128, 256) : sdesc(b, N * 16, 128);
    const long long t0 = clock64();
    if (mode == 2) {  // 8 MMAs in one asm block, alternating 2 accumulators, predicate set once
      const uint32_t d0 = tmem + 256, d1 = tmem + 256 + 128;
      for (int r = 0; r < reps; ++r)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t}\n" ::"r"(d0),
            "r"(d1), "l"(ad), "l"(bd), "r"(id));
    } else
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const uint32_t dst = tmem + 256 + (uint32_t)((g % nacc) * (256 / nacc));
        if (mode == 0) mma(dst, ad, bd, id, 1);
        else mma_ts(dst, tmem, bd, id, 1);
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_before();
  __syncthreads();
  if (tid < 32) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 512;
  for (int mode = 0; mode < 4; ++mode)
    for (int nacc : {1, 2, 4, 8})
      for (int N : {32, 64, 128, 256}) {
        if (N * nacc > 256 || (mode >= 2 && nacc != 2)) continue;
        bench<<<148, 128, 96 * 1024>>>(N, mode, 0, reps, nacc, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        const double cyc = s / 148 / (reps * 8.0);
        printf("%s A, %d accumulators, M=128 N=%3d K=16: %7.1f cycles/MMA (floor %5.1f)  %s\n", mode == 1 ? "TMEM" : (mode == 2 ? "smem/asm8" : (mode == 3 ? "smem/warp+elect" : "smem")),
               nacc, N, cyc, 128.0 * N / 256.0, cudaGetErrorString(e));
      }
  return 0;
}
