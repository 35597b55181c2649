/*
 * xlmimo_b200.h -- C-ABI of the B200-native Jac-PCG RZF precoding path.
 *
 * Drop-in boundary for the reference simulator's hot path
 * (/root/reference/pkg/src/xlmimo, pure Python/numpy).  The reference has no
 * FFI; its operator surface is the Python function set re-exported by
 * __init__.py:5-28.  Each entry point below replaces one (group of) those
 * functions for a BATCH of independent realizations; the Python mirror in
 * paper_2305_13925_b200/ binds them with ctypes.
 *
 * Conventions
 *  - dtype: XL_C64 = interleaved float2 (numpy complex64),
 *           XL_C128 = interleaved double2 (numpy complex128).
 *  - All matrices are C-order and batch-major: H[B][M][K] (rows = antennas,
 *    columns = users, exactly the reference layout), A/X[B][K][K].
 *  - All pointers are DEVICE pointers unless stated otherwise; calls are
 *    stream-ordered and asynchronous; no hidden allocation (caller passes a
 *    workspace sized by the matching *_workspace_bytes()).  One exception to
 *    "one stream": an xl_rzf call on K = 256 complex64 with B >= 1024 runs its
 *    chunks over the caller's stream and one internal stream (created once
 *    per host thread and device), forked from and joined back into `stream`
 *    with events -- still ordered on `stream` and CUDA-graph capturable.
 *  - Return value: XL_SUCCESS or an XL_ERR_* code (host-side argument errors
 *    map to the reference's ConfigurationError).  Numerical failures are
 *    reported per realization in status[B] (XL_STATUS_*), which the Python
 *    layer raises as the reference exception class.
 */
#ifndef XLMIMO_B200_H
#define XLMIMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* xl_stream_t; /* == cudaStream_t */

enum { XL_C64 = 0, XL_C128 = 1 };
enum { XL_JACPCG = 0, XL_CG = 1, XL_DIRECT = 2 };          /* precoder.py:109-115 */
enum { XL_JOR = 3, XL_GS = 4 };  /* stationary splittings, ITERATIVE_SOLVERS linsolve.py:310-315 */
enum { XL_TEXTBOOK = 0, XL_ALGORITHM = 1 };                /* linsolve.py:209-213 */

enum {
  XL_STATUS_OK = 0,
  XL_STATUS_NOT_HPD = 1,     /* curvature <= 0 with rz > 0: linsolve.py:240-242, 277-279 */
  XL_STATUS_SPLITTING = 2,   /* zero preconditioner diagonal: linsolve.py:205-208 */
  XL_STATUS_DEGENERATE = 3,  /* tr(F^H F) <= 0: precoder.py:66-68 */
  XL_STATUS_CHOLESKY = 4,    /* Cholesky breakdown -> NotHpdError: linsolve.py:113-116 */
  XL_STATUS_NO_VISIBLE = 5,  /* generator: no visible subarray (geometry.py:179-180) */
  XL_STATUS_RANGE = 6        /* fused c64 kernel: |H| dynamic range exceeds the fp16-split
                                scaling; re-run those realizations with xl_rzf_general */
};

enum {
  XL_SUCCESS = 0,
  XL_ERR_CONFIG = 1,       /* ConfigurationError: T<1, xi<=0, sigma2<=0, bad sizes */
  XL_ERR_CUDA = 2,         /* CUDA launch / runtime error (xl_last_error) */
  XL_ERR_UNSUPPORTED = 3,  /* shape outside the kernels' limits */
  XL_ERR_WORKSPACE = 4     /* workspace too small */
};

int xl_abi_version(void);
const char* xl_last_error(void);
/* Number of kernels this library has launched in the process so far
 * (benchmark accounting of "our" launches). */
uint64_t xl_launch_count(void);
/* Which tensor-core path serves the whole rzf call for (dtype, method, M, K):
 * 1 = tcgen05 (the fused kernel at K = 64 or K in {16, 32} with M K > 8192,
 * the streaming Gram / W + cluster Jac-PCG chain at K in {128, 256}),
 * 2 = warp-level mma.sync (complex64 K in {16, 32}, M % 32 == 0, M K <= 8192:
 * the small-K fused kernel), 3 = the same kernel with its Gram / W on tcgen05
 * (K = 32, M % 128 == 0; XL_SMALL_K_TC=0 selects 2), 0 = none (SIMT / DMMA). */
int xl_rzf_uses_tensor_cores(int dtype, int method, int32_t M, int32_t K);

/* Batched regularized Gram A_b = H_b^H H_b + xi_b I, Hermitian by
 * construction (lower triangle computed, mirrored, real diagonal).
 * Replaces gram_regularized (precoder.py:53-61).  xi_per_batch may be NULL
 * (then xi is used for every realization). */
int xl_gram(int dtype, const void* H, int64_t B, int32_t M, int32_t K,
            double xi, const double* xi_per_batch, void* A, xl_stream_t stream);

/* Batched HPD solve A_b X_b = S_b.
 * Replaces jacpcg_solve (linsolve.py:190-214; variant textbook -> 259-294,
 * algorithm -> 217-256), cg_solve (183-187) and direct_solve (109-119).
 *   S        [B][K][R] or NULL (identity right-hand sides, requires R == K)
 *   w0       [B][K][R] or NULL (zero initial guess, linsolve.py:78-79)
 *   precond  [B][K] real preconditioner diagonal or NULL (Re diag(A));
 *            precond_identity != 0 forces C = I.
 *   eps      < 0 means None (fixed-T mode); else stop when sqrt(trace) <= eps.
 *   X        [B][K][R]; iterations [B]; trace [B][T+1] or NULL
 *            (||A w_t - S||_F^2 / ||S||_F^2, trailing entries after an early
 *            stop are NaN); iterates [B][T][K][R] or NULL; status [B].
 * method == XL_DIRECT ignores T/variant/precond/w0/eps. */
size_t xl_solve_workspace_bytes(int dtype, int64_t B, int32_t K, int32_t R);
int xl_solve(int dtype, int method, int variant, const void* A, int64_t B,
             int32_t K, const void* S, int32_t R, const void* w0,
             const double* precond, int32_t precond_identity, int32_t T,
             double eps, void* X, int32_t* iterations, double* trace,
             void* iterates, int32_t* status, void* workspace,
             size_t ws_bytes, xl_stream_t stream);

/* Stationary iterative solvers on the same batched layout and workspace
 * (xl_solve_workspace_bytes):
 *   XL_JOR: w <- w + omega (s - P w) / diag(P)  -- replaces jor_solve (linsolve.py:154-176)
 *   XL_GS : (D + Lo) w' = s - Up w              -- replaces gs_solve  (linsolve.py:128-151)
 * A zero diagonal entry sets status XL_STATUS_SPLITTING (_check_diag :120-125);
 * omega <= 0 or T < 1 -> XL_ERR_CONFIG (ConfigurationError).  S, w0, eps, X,
 * iterations, trace, iterates, status as in xl_solve. */
int xl_solve_stationary(int dtype, int method, const void* A, int64_t B, int32_t K,
                        const void* S, int32_t R, const void* w0, double omega,
                        int32_t T, double eps, void* X, int32_t* iterations,
                        double* trace, void* iterates, int32_t* status,
                        void* workspace, size_t ws_bytes, xl_stream_t stream);

/* The fused hot path, per realization b:
 *   A = H^H H + xi I; X ~= A^{-1} (Jac-PCG / CG with T iterations, identity
 *   RHS, w0 = 0, or Cholesky for XL_DIRECT); F = H X;
 *   beta = sqrt(power / ||F||_F^2); W = beta F;
 *   B = H^H W; gamma_k = |B_kk|^2 / (sum_j |B_kj|^2 - |B_kk|^2 + sigma2);
 *   sum_se = sum_k log2(1 + gamma_k).
 * Replaces rzf_iterative / rzf_direct (precoder.py:73-91), _power_scale
 * (64-70) and sinr_eq9 (metrics.py:47-58) on one full-array block.
 *   W [B][M][K]; F [B][M][K] or NULL; beta [B]; gamma [B][K] (double) or NULL;
 *   sum_se [B]; X [B][K][K] or NULL; status [B]. */
size_t xl_rzf_workspace_bytes(int dtype, int method, int64_t B, int32_t M,
                              int32_t K);
int xl_rzf(int dtype, int method, int variant, const void* H, int64_t B,
           int32_t M, int32_t K, double xi, const double* xi_per_batch,
           double power, int32_t T, double sigma2, void* W, void* F,
           double* beta, double* gamma, double* sum_se, void* X,
           int32_t* status, void* workspace, size_t ws_bytes,
           xl_stream_t stream);

/* xl_rzf with the solver telemetry of SolverOutcome (linsolve.py:60-68):
 *   iterations [B] (T for Jac-PCG / CG in fixed-T mode, 0 for XL_DIRECT);
 *   trace [B][T+1] or NULL: the squared relative least-squares error
 *   ||A x_t - I||_F^2 / ||I||_F^2 after t = 0..T iterations (_ls_error,
 *   linsolve.py:89-91; XL_DIRECT: one entry).
 * The trace_opt / iterations outputs of SURVEY.md section 8(b)'s xl_rzf; runs
 * on the general kernels (the SIMT solver records the trace) with the
 * workspace of xl_rzf_general_workspace_bytes.  Same status codes as xl_rzf. */
int xl_rzf_traced(int dtype, int method, int variant, const void* H, int64_t B,
                  int32_t M, int32_t K, double xi, const double* xi_per_batch,
                  double power, int32_t T, double sigma2, void* W, void* F,
                  double* beta, double* gamma, double* sum_se, void* X,
                  int32_t* iterations, double* trace, int32_t* status,
                  void* workspace, size_t ws_bytes, xl_stream_t stream);

/* Second half of the hot path for a given solution X ~= A^{-1} (e.g. from
 * xl_solve with an eps stop): F = H X, beta = sqrt(power/||F||_F^2),
 * W = beta F, SINR/SE.  precoder.py:88-91 + 64-70, metrics.py:47-58. */
size_t xl_apply_precoder_workspace_bytes(int dtype, int64_t B, int32_t M, int32_t K);
int xl_apply_precoder(int dtype, const void* H, const void* X, int64_t B, int32_t M,
                      int32_t K, double power, double sigma2, void* W, void* F,
                      double* beta, double* gamma, double* sum_se, int32_t* status,
                      void* workspace, size_t ws_bytes, xl_stream_t stream);

/* Same contract as xl_rzf, always on the general (SIMT) kernels; the
 * fallback for XL_STATUS_RANGE realizations and a cross-check of the fused
 * tensor-core path. */
size_t xl_rzf_general_workspace_bytes(int dtype, int method, int64_t B, int32_t M,
                                      int32_t K);
int xl_rzf_general(int dtype, int method, int variant, const void* H, int64_t B,
                   int32_t M, int32_t K, double xi, const double* xi_per_batch,
                   double power, int32_t T, double sigma2, void* W, void* F,
                   double* beta, double* gamma, double* sum_se, void* X,
                   int32_t* status, void* workspace, size_t ws_bytes,
                   xl_stream_t stream);
/* Test hook: when non-NULL, the fused kernel also writes the regularized Gram
 * A[B][K][K] (complex64) of every realization it processes. */
void xl_debug_set_gram_out(void* A);
/* Development hook: when non-NULL, the K = 256 cluster solver writes clock64
 * stamps of cluster 0 / CTA 0 (phase boundaries) into buf[0..255]. */
void xl_debug_lk_trace(void* buf);

/* Per-user SINR/SE of an arbitrary precoder G on one full-array block:
 * sinr_eq9 (metrics.py:47-58) with coupling B = H^H G (metrics.py:35-44).
 * gamma/se [B][K] double, sum_se [B]. */
size_t xl_sinr_workspace_bytes(int dtype, int64_t B, int32_t K);
int xl_sinr(int dtype, const void* H, const void* G, int64_t B, int32_t M,
            int32_t K, double sigma2, double* gamma, double* se,
            double* sum_se, void* workspace, size_t ws_bytes,
            xl_stream_t stream);

/* On-device channel batch (BASELINE model; recipe of scenario.py:85-96):
 * H[b] for global realization indices first .. first+B-1, M = S*Ms.
 * Rsqrt [Ms][Ms] device doubles (psd_sqrt of the exponential correlation,
 * channel.py:33-53); gain = 10^(beta_dB/10) / beta_bar (beta_bar = 1 keeps
 * the raw path loss).  Philox4x32-10 counter map documented in DESIGN.md. */
int xl_channel_generate(int dtype, uint64_t seed, int64_t first, int64_t B,
                        int32_t S, int32_t Ms, int32_t K, double p,
                        const double* Rsqrt, double beta_bar, double dmin,
                        double dmax, void* H, int32_t* status,
                        xl_stream_t stream);

/* Ergodic-SE partials for sum_se (metrics.py:61-68): for every chunk c of
 * `chunk` consecutive realizations, partials[c] = {sum x, sum x^2, n} in
 * index order (deterministic, combined across ranks in chunk order). */
int xl_se_partials(const double* sum_se, int64_t B, int64_t chunk,
                   double* partials, xl_stream_t stream);

/* mean_sem[0..1] = {mean, SEM (ddof = 1)} of the realizations behind
 * n_chunks ordered partials (as produced by xl_se_partials, possibly
 * gathered over ranks), summed in chunk order on the device: the tail of
 * sum_se's mean/SEM (metrics.py:61-68) without a host round trip. */
int xl_se_combine(const double* partials, int64_t n_chunks, double* mean_sem,
                  xl_stream_t stream);

/* BER detection chain of ber_montecarlo (metrics.py:124-140) for a batch of
 * channel draws: Y = Bc s + n with s = QPSK(bits) ((1-2b0) + j(1-2b1))/sqrt(2)
 * (metrics.py:73-77), genie scaling by diag(Bc) with zero gains replaced by 1,
 * hard decisions b = (Re < 0, Im < 0) (metrics.py:80-83), and the number of
 * bit errors per draw.  Bc [B][K][K] (coupling, e.g. sinr's B = H^H G);
 * bits [B][K][nsym][2] int8 in {0,1}; noise [B][K][nsym]; errors [B] int64
 * (overwritten). */
int xl_ber_errors(int dtype, const void* Bc, const int8_t* bits, const void* noise,
                  int64_t B, int32_t K, int32_t nsym, int64_t* errors,
                  xl_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* XLMIMO_B200_H */
