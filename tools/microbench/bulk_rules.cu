// Per-SM fill rate of cp.async.bulk (global -> shared) vs piece size, number
// of issuing lanes and copies in flight.  Each CTA (one per SM) streams 2 MiB
// from its own L2-resident 512 KiB window: `lanes` lanes each keep `depth`
// copies of `piece` bytes in flight (own mbarrier per lane and slot).
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

namespace t {
#include "../../paper_2305_13925_b200/csrc/tc_ptx.cuh"
}
using namespace t;

__global__ void __launch_bounds__(32, 1) fill(const uint8_t* src, int piece, int lanes, int depth, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32 * 8];
  const int l = threadIdx.x;
  if (l < lanes)
    for (int d = 0; d < depth; ++d) mbar_init(&bar[l * 8 + d], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const size_t span = 512 * 1024;
  const uint8_t* base = src + (size_t)blockIdx.x * span;
  const uint64_t pol = policy_evict_normal();
  const int per_lane = (int)((4 * span) / piece / lanes);
  const long long t0 = clock64();
  if (l < lanes) {
    for (int g = 0; g < per_lane + depth; ++g) {
      const int d = g % depth;
      if (g >= depth) mbar_wait(&bar[l * 8 + d], ((g - depth) / depth) & 1);
      if (g < per_lane) {
        mbar_expect_tx(&bar[l * 8 + d], piece);
        uint8_t* dst = sm + (size_t)(l * depth + d) * piece;
        bulk_g2s(dst, base + ((size_t)(g * lanes + l) * piece) % span, piece, &bar[l * 8 + d], pol);
      }
    }
  }
  __syncwarp();
  if (l == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t* buf;
  cudaMalloc(&buf, (size_t)512 * 1024 * 148);
  cudaMemset(buf, 1, (size_t)512 * 1024 * 148);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int piece : {2048, 4096, 8192, 16384, 32768})
    for (int lanes : {1, 2, 4, 8, 16})
      for (int depth : {1, 2, 4}) {
        if ((size_t)piece * lanes * depth > 192 * 1024) continue;
        fill<<<148, 32, 200 * 1024>>>(buf, piece, lanes, depth, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = fmax(mx, (double)h[i]);
        printf("piece %6d B lanes %2d depth %d (in flight %4d KiB): %6.1f B/cycle/SM %s\n", piece, lanes, depth,
               piece * lanes * depth / 1024, (double)(4 * 512 * 1024) / mx, e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
