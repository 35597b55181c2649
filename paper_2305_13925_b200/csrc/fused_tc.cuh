// Fused tcgen05 precoder (complex64 hot shapes).  See fused_tc.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace xl {
bool fused_supported(int dtype, int method, int M, int K);
size_t fused_ws_bytes(int dtype, int method, int64_t B, int M, int K);
int launch_fused(int dtype, int method, int variant, const void* H, int64_t B, int M, int K,
                 double xi, const double* xi_per_batch, double power, int T, double sigma2,
                 void* W, void* F, double* beta, double* gamma, double* sum_se, void* X,
                 int32_t* status, void* ws, size_t ws_bytes, void* dbg_gram, cudaStream_t st);
}  // namespace xl
