// Tensor-core products of the general precoder path for large K (the fused
// tcgen05 kernel covers K <= 64): the batched Gram A = H^H H + xi I and the
// precoder W = beta H X.
//
// complex64 -> 3xTF32.  A split kernel writes, per antenna row m of the real
// view Z = [Re h, Im h] (M x 2K), the row [Zh | Zl] with Zh = tf32(Z) (round to
// nearest, exact in TF32) and Zl = Z - Zh (exact in fp32); the products run as
// plain TF32 GEMMs with fp32 accumulation:
//   Gram: U = Zh^T Zh + 2 Zh^T Zl, G = (U + U^T) / 2 = Zh^T Zh + Zh^T Zl + Zl^T Zh
//   W   : W = Z Xe with Xe the real embedding of beta X, split the same way:
//         W = [Xeh ; Xeh]^T-stacked [Zh | Zl] + Zl-free Xel term
//         (= Zh Xeh + Zl Xeh + Zh Xel, two GEMMs)
// ~21 significant bits per product, the same class as the fused kernel's
// 3xFP16 but with TF32's 8-bit exponent (no pre-scaling).
// complex128 -> ZGEMM (FP64 tensor cores).
//
// The GEMMs are plain library GEMMs (cuBLAS, strided batched, caller-provided
// cuBLAS workspace); the split / embedding / Gram-extraction kernels are ours.
// Reference ops replaced: precoder.py:59-60 (H^H H + xi I, symmetrised) and
// precoder.py:88-91 + 64-70 (F = H X, G = beta F).
#include <cublas_v2.h>
#include <mutex>

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {

namespace {

constexpr size_t CUBLAS_WS = 32u << 20;  // cuBLAS workspace carved from the caller's

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

cublasHandle_t handle_for_device() {
  static std::mutex mu;
  static cublasHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!handles[dev]) {
    if (cublasCreate(&handles[dev]) != CUBLAS_STATUS_SUCCESS) return nullptr;
  }
  return handles[dev];
}

int cublas_check(cublasStatus_t s, const char* what) {  // library launches: not counted as ours
  if (s == CUBLAS_STATUS_SUCCESS) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return XL_SUCCESS;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return XL_ERR_CUDA;
  }
  set_error("%s: cuBLAS status %d", what, (int)s);
  return XL_ERR_CUDA;
}

__device__ __forceinline__ float tf32_rn(float x) {
  // round to nearest (ties away) onto the 10-bit TF32 mantissa; finite inputs
  uint32_t u = __float_as_uint(x);
  u = (u + 0x1000u) & 0xffffe000u;
  return __uint_as_float(u);
}

// Z (nrow x n2, row-major) -> S (nrow x 2 n2): row [Zh | Zl]
__global__ void split_rows_kernel(const float4* __restrict__ Z, float4* __restrict__ S, int64_t nrow, int n2) {
  const int q = n2 / 4;
  const int64_t total = nrow * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / q;
    const int c = (int)(e % q);
    const float4 x = Z[e];
    float4 h, l;
    h.x = tf32_rn(x.x); h.y = tf32_rn(x.y); h.z = tf32_rn(x.z); h.w = tf32_rn(x.w);
    l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
    S[r * 2 * q + c] = h;
    S[r * 2 * q + q + c] = l;
  }
}

// U [b] (n2 x n2) -> A[b] (K x K complex): G = (U + U^T)/2,
// Re A_ij = G[2i][2j] + G[2i+1][2j+1], Im A_ij = G[2i][2j+1] - G[2i+1][2j], + xi on the
// diagonal.  Exactly Hermitian by construction (real diagonal).
__global__ void gram_extract_kernel(const float* __restrict__ U, float2* __restrict__ A, int K,
                                    const double* __restrict__ xi_b, double xi) {
  const int64_t b = blockIdx.y;
  const int n2 = 2 * K;
  const float* u = U + b * (int64_t)n2 * n2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * K; e += gridDim.x * blockDim.x) {
    const int i = e / K, j = e % K;
    auto g = [&](int r, int c) { return 0.5f * (u[(int64_t)r * n2 + c] + u[(int64_t)c * n2 + r]); };
    float re = g(2 * i, 2 * j) + g(2 * i + 1, 2 * j + 1);
    float im = g(2 * i, 2 * j + 1) - g(2 * i + 1, 2 * j);
    if (i == j) {
      re = (float)((double)re + (xi_b ? xi_b[b] : xi));
      im = 0.0f;
    }
    A[b * (int64_t)K * K + e] = make_float2(re, im);
  }
}

// beta X (K x K complex) -> the split real embedding as the GEMM's A operands,
// column-major n2 x n2 views of row-major Xe (i.e. Xe^T):
//   E1 (n2 x 2 n2) = [Xeh^T | Xeh^T]  (pairs with S's [Zh ; Zl] rows)
//   E2 (n2 x n2)   = Xel^T            (pairs with Zh)
// Xe[2i][2j] = xr, Xe[2i][2j+1] = xi, Xe[2i+1][2j] = -xi, Xe[2i+1][2j+1] = xr.
__global__ void embed_x_kernel(const float2* __restrict__ X, const double* __restrict__ beta, float* __restrict__ E1,
                               float* __restrict__ E2, int K) {
  const int64_t b = blockIdx.y;
  const int n2 = 2 * K;
  const float sc = (float)beta[b];
  float* e1 = E1 + b * (int64_t)n2 * 2 * n2;
  float* e2 = E2 + b * (int64_t)n2 * n2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2 * n2; e += gridDim.x * blockDim.x) {
    const int r = e / n2, c = e % n2;  // Xe[r][c]
    const float2 x = X[b * (int64_t)K * K + (r / 2) * K + (c / 2)];
    const float xr = x.x * sc, xi = x.y * sc;
    const float v = (r & 1) == 0 ? ((c & 1) == 0 ? xr : xi) : ((c & 1) == 0 ? -xi : xr);
    const float h = tf32_rn(v), l = v - h;
    // column-major (n2 rows) view of row-major Xe: element (c, r) at r * n2 + c
    e1[(int64_t)r * n2 + c] = h;
    e1[(int64_t)(n2 + r) * n2 + c] = h;
    e2[(int64_t)r * n2 + c] = l;
  }
}

__global__ void scale_copy_kernel(const float2* __restrict__ W, float2* __restrict__ F, const double* __restrict__ beta,
                                  int64_t per, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const float s = (float)(1.0 / beta[e / per]);
    const float2 w = W[e];
    F[e] = make_float2(w.x * s, w.y * s);
  }
}

// W <- beta W (and F <- the unscaled product when requested), complex128
__global__ void scale_c128_kernel(double2* __restrict__ W, double2* __restrict__ F, const double* __restrict__ beta,
                                  int64_t per, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const double s = beta[e / per];
    const double2 w = W[e];
    if (F) F[e] = w;
    W[e] = make_double2(w.x * s, w.y * s);
  }
}

__global__ void herm_add_kernel(double2* __restrict__ A, int K, const double* __restrict__ xi_b, double xi) {
  // (P + P^H)/2 + xi I on the ZGEMM result (precoder.py:59-60)
  const int64_t b = blockIdx.y;
  double2* a = A + b * (int64_t)K * K;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * K; e += gridDim.x * blockDim.x) {
    const int i = e / K, j = e % K;
    if (j > i) continue;
    const double2 p = a[(int64_t)i * K + j], q = a[(int64_t)j * K + i];
    if (i == j) {
      a[e] = make_double2(p.x + (xi_b ? xi_b[b] : xi), 0.0);
    } else {
      const double re = 0.5 * (p.x + q.x), im = 0.5 * (p.y - q.y);
      a[(int64_t)i * K + j] = make_double2(re, im);
      a[(int64_t)j * K + i] = make_double2(re, -im);
    }
  }
}

unsigned grid_for(int64_t n, int t) {
  int64_t g = (n + t - 1) / t;
  return (unsigned)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

bool tc_general_supported(int dtype, int M, int K) {
  (void)M;
  return K >= 96 && (dtype == XL_C128 || (2 * K) % 4 == 0);
}

size_t tc_gram_ws_bytes(int dtype, int64_t Bc, int M, int K) {
  if (dtype == XL_C128) return CUBLAS_WS;
  const size_t n2 = 2 * (size_t)K;
  return CUBLAS_WS + align_up((size_t)Bc * M * 2 * n2 * 4) + align_up((size_t)Bc * n2 * n2 * 4) +
         align_up((size_t)Bc * n2 * 3 * n2 * 4);
}

// S = split(H) for Bc realizations, then A = H^H H + xi I.  The split rows stay in
// the workspace for tc_apply on the same realizations.
int tc_gram(int dtype, const void* H, int64_t Bc, int M, int K, const double* xi_b, double xi, void* A,
            void* ws, cudaStream_t st) {
  cublasHandle_t h = handle_for_device();
  if (!h) { set_error("cublasCreate failed"); return XL_ERR_CUDA; }
  cublasSetStream(h, st);
  char* p = (char*)ws;
  cublasSetWorkspace(h, p, CUBLAS_WS);
  p += CUBLAS_WS;
  if (dtype == XL_C128) {
    const cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    // column-major C = H_cm H_cm^H (K x K) has the memory of row-major H^H H
    int e = cublas_check(cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_C, K, K, M, &one,
                                                   (const cuDoubleComplex*)H, K, (long long)M * K,
                                                   (const cuDoubleComplex*)H, K, (long long)M * K, &zero,
                                                   (cuDoubleComplex*)A, K, (long long)K * K, (int)Bc),
                         "tc gram zgemm");
    if (e) return e;
    const unsigned gk = grid_for((int64_t)K * K, 256);
    herm_add_kernel<<<dim3(gk > 64 ? 64 : gk, (unsigned)Bc), 256, 0, st>>>((double2*)A, K, xi_b, xi);
    return check_launch("tc herm");
  }
  const int n2 = 2 * K;
  float* S = (float*)p;
  p += align_up((size_t)Bc * M * 2 * n2 * 4);
  float* U = (float*)p;
  const int64_t nrow = Bc * (int64_t)M;
  split_rows_kernel<<<grid_for(nrow * n2 / 4, 256), 256, 0, st>>>((const float4*)H, (float4*)S, nrow, n2);
  if (int e = check_launch("tc split")) return e;
  const float one = 1.0f, two = 2.0f, zero = 0.0f;
  const long long sS = (long long)M * 2 * n2, sU = (long long)n2 * n2;
  // U = Zh Zh^T (col-major: S rows 0..n2-1 of each column, ld 2 n2), then += 2 Zh Zl^T
  int e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_T, n2, n2, M, &one, S, CUDA_R_32F, 2 * n2, sS,
                                                  S, CUDA_R_32F, 2 * n2, sS, &zero, U, CUDA_R_32F, n2, sU, (int)Bc,
                                                  CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                       "tc gram hh");
  if (e) return e;
  e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_T, n2, n2, M, &two, S, CUDA_R_32F, 2 * n2, sS,
                                              S + n2, CUDA_R_32F, 2 * n2, sS, &one, U, CUDA_R_32F, n2, sU, (int)Bc,
                                              CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                   "tc gram hl");
  if (e) return e;
  unsigned gx = grid_for((int64_t)K * K, 256);
  gram_extract_kernel<<<dim3(gx > 64 ? 64 : gx, (unsigned)Bc), 256, 0, st>>>(U, (float2*)A, K, xi_b, xi);
  return check_launch("tc gram extract");
}

// W = beta H X for Bc realizations; their split rows are in ws from tc_gram
// unless resplit; F = W / beta when requested.
int tc_apply(int dtype, const void* H, const void* X, const double* beta, int64_t Bc, int M, int K, void* W,
             void* F, void* ws, cudaStream_t st, bool resplit) {
  cublasHandle_t h = handle_for_device();
  if (!h) { set_error("cublasCreate failed"); return XL_ERR_CUDA; }
  cublasSetStream(h, st);
  char* p = (char*)ws;
  cublasSetWorkspace(h, p, CUBLAS_WS);
  p += CUBLAS_WS;
  if (dtype == XL_C128) {
    // W_cm (K x M) = X_mem (col-major view = X^T) . H_cm: the memory of row-major H X;
    // beta applied by the epilogue kernel below
    const cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    int e = cublas_check(cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, K, M, K, &one,
                                                   (const cuDoubleComplex*)X, K, (long long)K * K,
                                                   (const cuDoubleComplex*)H, K, (long long)M * K, &zero,
                                                   (cuDoubleComplex*)W, K, (long long)M * K, (int)Bc),
                         "tc apply zgemm");
    if (e) return e;
    const int64_t per = (int64_t)M * K, total = Bc * per;
    scale_c128_kernel<<<grid_for(total, 256), 256, 0, st>>>((double2*)W, (double2*)F, beta, per, total);
    return check_launch("tc scale");
  }
  const int n2 = 2 * K;
  float* S = (float*)p;
  p += align_up((size_t)Bc * M * 2 * n2 * 4);
  p += align_up((size_t)Bc * n2 * n2 * 4);  // U (unused here)
  float* E1 = (float*)p;
  float* E2 = E1 + (size_t)Bc * n2 * 2 * n2;
  if (resplit) {
    const int64_t nrow = Bc * (int64_t)M;
    split_rows_kernel<<<grid_for(nrow * n2 / 4, 256), 256, 0, st>>>((const float4*)H, (float4*)S, nrow, n2);
    if (int e = check_launch("tc split")) return e;
  }
  unsigned gx = grid_for((int64_t)n2 * n2, 256);
  embed_x_kernel<<<dim3(gx > 64 ? 64 : gx, (unsigned)Bc), 256, 0, st>>>((const float2*)X, beta, E1, E2, K);
  if (int e = check_launch("tc embed")) return e;
  const float one = 1.0f, zero = 0.0f;
  const long long sS = (long long)M * 2 * n2, sW = (long long)M * n2;
  // W_cm (n2 x M) = E1 (n2 x 2n2) . S (2n2 x M)  +  E2 (n2 x n2) . Zh (n2 x M, ld 2 n2)
  int e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, M, 2 * n2, &one, E1, CUDA_R_32F, n2,
                                                  (long long)n2 * 2 * n2, S, CUDA_R_32F, 2 * n2, sS, &zero, W,
                                                  CUDA_R_32F, n2, sW, (int)Bc, CUBLAS_COMPUTE_32F_FAST_TF32,
                                                  CUBLAS_GEMM_DEFAULT),
                       "tc apply hh+lh");
  if (e) return e;
  e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, M, n2, &one, E2, CUDA_R_32F, n2,
                                              (long long)n2 * n2, S, CUDA_R_32F, 2 * n2, sS, &one, W, CUDA_R_32F, n2,
                                              sW, (int)Bc, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                   "tc apply hl");
  if (e) return e;
  if (F) {
    const int64_t per = (int64_t)M * K, total = Bc * per;
    scale_copy_kernel<<<grid_for(total, 256), 256, 0, st>>>((const float2*)W, (float2*)F, beta, per, total);
    return check_launch("tc F");
  }
  return XL_SUCCESS;
}

}  // namespace xl
