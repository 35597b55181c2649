// Host-side launchers of the SIMT (general-shape / complex128) kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace xl {

enum { EPI_STORE = 0, EPI_GRAM = 1, EPI_FNORM = 2, EPI_GXF = 3, EPI_BSCALE = 4 };

template <typename R>
int launch_cgemm(bool conjA, int epi, const void* A, int64_t sA, int lda,
                 const void* Bm, int64_t sB, int ldb, void* Cm, int64_t sC,
                 int ldc, int64_t batch, int m, int n, int k,
                 const double* diag_add, double diag_scalar, double* partial,
                 cudaStream_t st);
int gemm_tiles(int m, int n);

template <typename R>
int launch_beta_scale(void* W, void* F, int64_t B, int64_t per, const double* partial,
                      int nparts, double power, double* beta, int32_t* status,
                      cudaStream_t st);
template <typename R>
int launch_sinr(const void* Bc, int64_t B, int K, double sigma2, double* gamma,
                double* se, double* sum_se, cudaStream_t st, const double* bscale = nullptr);
int launch_beta_from_partials(int64_t B, const double* partial, int nparts, double power, double* beta,
                              int32_t* status, cudaStream_t st);
int launch_se_partials(const double* s, int64_t B, int64_t chunk, double* out, cudaStream_t st);
int launch_se_combine(const double* parts, int64_t nc, double* out, cudaStream_t st);

// PCG / CG / Jac-PCG (linsolve.py:183-294) and Cholesky (linsolve.py:109-119).
struct SolveArgs {
  int method, variant;
  const void* A; int64_t B; int K;
  const void* S; int R;          // S == nullptr -> identity (R == K)
  const void* w0;                // nullable
  const double* precond;         // nullable -> Re diag(A)
  int precond_identity;
  int T; double eps;             // eps < 0 -> None
  void* X; int32_t* iterations; double* trace; void* iterates; int32_t* status;
  void* ws; size_t ws_bytes;
  double omega = 0.5;            // XL_JOR relaxation
};
template <typename R> size_t solve_ws_bytes(int64_t B, int K, int Rcols);
template <typename R> int launch_solve(const SolveArgs& a, cudaStream_t st);

// gemm_tc.cu: tensor-core Gram / W for the general path at large K (3xTF32 c64, ZGEMM c128)
bool tc_general_supported(int dtype, int M, int K);
size_t tc_gram_ws_bytes(int dtype, int64_t Bc, int M, int K);
int tc_gram(int dtype, const void* H, int64_t Bc, int M, int K, const double* xi_b, double xi, void* A,
            void* ws, cudaStream_t st);
int tc_apply(int dtype, const void* H, const void* X, const double* beta, int64_t Bc, int M, int K, void* W,
             void* F, void* ws, cudaStream_t st, bool resplit);

size_t tc_pcg_ws_bytes(int64_t B, int K);
bool tc_pcg_supported(int K);
size_t tc_pcg64_ws_bytes(int64_t B, int K);
bool tc_pcg64_supported(int K);
int tc_pcg64(int method, int variant, const void* A, int64_t B, int K, int T, void* X, int32_t* status, void* cws,
             void* bufs, cudaStream_t st);
int tc_gx64(const void* A, const double* xi_b, double xi, int64_t B, int K, void* GX, double* part, void* cws,
            void* bufs, cudaStream_t st);
int tc_gx(const double* xi_b, double xi, int64_t B, int K, void* GX, double* part, void* cws, void* bufs,
          cudaStream_t st);
// stream_tc.cu: streaming tcgen05 Gram / W for K = 128 complex64 (M % 64 == 0)
bool stc_supported(int dtype, int M, int K);
int stc_gram(const void* H, int64_t B, int M, int K, double xi, const double* xi_b, float* sz, void* A, int* rflag,
             cudaStream_t st);
int stc_apply(const void* H, const void* X, const double* beta, const float* sz, int64_t B, int M, int K, void* W,
              void* F, cudaStream_t st);
int tc_gram_extract(const float* U, int64_t Bc, int K, const double* xi_b, double xi, void* A, cudaStream_t st);
size_t tc_cublas_ws_bytes();
// cluster_pcg.cu: fused 2-CTA-cluster Jac-PCG / CG + GX for K = 128 (complex64)
bool cpcg_supported(int K);
int cpcg_solve(int method, int variant, const void* A, int64_t B, int K, int T, double xi, const double* xi_b,
               void* X, void* GX, double* part, int32_t* status, cudaStream_t st);
int tc_pcg(int method, int variant, const void* A, int64_t B, int K, int T, void* X, int32_t* status, void* cws,
           void* bufs, cudaStream_t st);

// large_k.cu: K = 256 complex64 -- streaming tcgen05 Gram / W and the 8-CTA cluster Jac-PCG
bool lk_supported(int dtype, int M, int K);
size_t lk_ws_bytes(int64_t B);
// per-realization scales / range flags / exact maxima, then the solver's cluster slots
struct LkScratch {
  float* sz;
  int* rflag;
  unsigned* zmax;
  uint8_t* slots;
};
LkScratch lk_scratch(void* ws, int64_t B);
int lk_gram(const void* H, int64_t B, int M, double xi, const double* xi_b, void* A, float* sz, int* rflag,
            unsigned* zmax, cudaStream_t st);
int lk_solve(int method, int variant, const void* A, int64_t B, int T, double xi, const double* xi_b, void* X,
             void* GX, double* part, int32_t* status, uint8_t* slots, cudaStream_t st);
void lk_debug_trace(void* buf);
// SINR / sum-SE from the K = 256 solver's partials (written into its GX buffer)
int lk_sinr(const void* GX, const double* beta, int64_t B, double sigma2, double* gamma, double* sum_se,
            cudaStream_t st);
int lk_apply(const void* H, const void* X, const double* beta, int64_t B, int M, void* W, void* F,
             const unsigned* zmax, const float* xmax, cudaStream_t st);
// the solver's per-column max |X| (in its GX buffer, after the SINR partials)
float* lk_xmax(void* GX, int64_t B);

// dmma.cu: batched complex128 GEMM on the FP64 tensor cores (row-major;
// opA 0 = N, 1 = conjugate transpose; opB 0 = N, 1 = transpose; epi 0 store,
// 1 = beta scale (+ unscaled copy F), 2 = Hermitian lower tiles + mirror + xi I)
int zgemm_dmma(int opA, const void* A, int64_t sA, int lda, int opB, const void* B, int64_t sB, int ldb, void* C,
               int64_t sC, int ldc, int M, int N, int K, int64_t batch, int epi, const double* beta, void* F,
               const double* xi_b, double xi, cudaStream_t st);

// fused_c128.cu: one CTA per realization, whole chain on chip, DMMA products (K in {16, 32})
bool fc128_supported(int dtype, int method, int M, int K);
int fc128_rzf(int method, int variant, const void* H, int64_t B, int M, int K, double xi, const double* xi_b,
              double power, int T, double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
              void* X, int32_t* status, cudaStream_t st);

// fused_c64s.cu: one CTA per realization (two per SM), Gram / W on mma.sync (3xFP16), fp32 SIMT solve
bool fc64s_supported(int dtype, int method, int M, int K);
bool fc64s_uses_tcgen05(int M, int K);
int fc64s_rzf(int method, int variant, const void* H, int64_t B, int M, int K, double xi, const double* xi_b,
              double power, int T, double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
              void* X, int32_t* status, cudaStream_t st);

int launch_ber(int dtype, const void* Bc, const int8_t* bits, const void* noise, int64_t B, int K,
               int nsym, int64_t* errors, cudaStream_t st);

int launch_channel(int dtype, uint64_t seed, int64_t first, int64_t B, int S, int Ms,
                   int K, double p, const double* Rsqrt, double gain_scale, double dmin,
                   double dmax, void* H, int32_t* status, cudaStream_t st);

}  // namespace xl
