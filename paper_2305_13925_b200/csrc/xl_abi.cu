// extern "C" boundary of libxlmimo_b200.so (declared in include/xlmimo_b200.h).
//
// Host-side argument validation mirrors the reference's ConfigurationError
// checks (precoder.py:55-56, 86-87; linsolve.py:209-210, 260-261;
// metrics.py:49-50) and returns XL_ERR_CONFIG before anything is launched.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "xl_common.cuh"
#include "simt_kernels.cuh"
#include "fused_tc.cuh"

namespace xl {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return XL_ERR_CUDA;
  }
  return XL_SUCCESS;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t csize(int dtype) { return dtype == XL_C64 ? 8 : 16; }

static int check_dtype(int dtype) {
  if (dtype != XL_C64 && dtype != XL_C128) { set_error("unknown dtype %d", dtype); return XL_ERR_CONFIG; }
  return XL_SUCCESS;
}

// F = H X (+ per-tile ||F||^2) -> beta, W = beta F -> B = H^H W -> SINR/SE.
static int apply_precoder(int dtype, const void* H, const void* X, int64_t B, int M, int K,
                          double power, double sigma2, void* W, void* F, double* beta,
                          double* gamma, double* sum_se, int32_t* status, double* part,
                          void* Bc, cudaStream_t st) {
  int64_t sH = (int64_t)M * K, sK = (int64_t)K * K;
  const int nparts = gemm_tiles(M, K);
  int e;
  if (dtype == XL_C64) {
    if ((e = launch_cgemm<float>(false, EPI_FNORM, H, sH, K, X, sK, K, W, sH, K, B, M, K, K, nullptr, 0, part, st))) return e;
    if ((e = launch_beta_scale<float>(W, F, B, sH, part, nparts, power, beta, status, st))) return e;
    if ((e = launch_cgemm<float>(true, EPI_STORE, H, sH, K, W, sH, K, Bc, sK, K, B, K, K, M, nullptr, 0, nullptr, st))) return e;
    return launch_sinr<float>(Bc, B, K, sigma2, gamma, nullptr, sum_se, st);
  }
  if ((e = launch_cgemm<double>(false, EPI_FNORM, H, sH, K, X, sK, K, W, sH, K, B, M, K, K, nullptr, 0, part, st))) return e;
  if ((e = launch_beta_scale<double>(W, F, B, sH, part, nparts, power, beta, status, st))) return e;
  if ((e = launch_cgemm<double>(true, EPI_STORE, H, sH, K, W, sH, K, Bc, sK, K, B, K, K, M, nullptr, 0, nullptr, st))) return e;
  return launch_sinr<double>(Bc, B, K, sigma2, gamma, nullptr, sum_se, st);
}

}  // namespace xl

using namespace xl;

extern "C" {

int xl_abi_version(void) { return 1; }
uint64_t xl_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }
const char* xl_last_error(void) { return g_err; }

int xl_rzf_uses_tensor_cores(int dtype, int method, int32_t M, int32_t K) {
  // small-K kernel (fused_c64s.cu): 3 = tcgen05 Gram / W + mma.sync solve, 2 = all mma.sync
  if (fc64s_supported(dtype, method, M, K)) return fc64s_uses_tcgen05(M, K) ? 3 : 2;
  if (fused_supported(dtype, method, M, K)) return 1;
  // K = 256: streaming tcgen05 Gram / W + the 8-CTA cluster Jac-PCG / CG
  if (method != XL_DIRECT && lk_supported(dtype, M, K)) return 1;
  // K = 128: streaming tcgen05 Gram / W + the cluster Jac-PCG / CG
  return (method != XL_DIRECT && stc_supported(dtype, M, K) && cpcg_supported(K)) ? 1 : 0;
}

int xl_gram(int dtype, const void* H, int64_t B, int32_t M, int32_t K, double xi,
            const double* xi_per_batch, void* A, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (!xi_per_batch && !(xi > 0)) { set_error("regularization xi must be positive, got %g", xi); return XL_ERR_CONFIG; }
  if (M < 1 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t sH = (int64_t)M * K, sA = (int64_t)K * K;
  if (dtype == XL_C64)
    return launch_cgemm<float>(true, EPI_GRAM, H, sH, K, H, sH, K, A, sA, K, B, K, K, M, xi_per_batch, xi, nullptr, st);
  return launch_cgemm<double>(true, EPI_GRAM, H, sH, K, H, sH, K, A, sA, K, B, K, K, M, xi_per_batch, xi, nullptr, st);
}

size_t xl_solve_workspace_bytes(int dtype, int64_t B, int32_t K, int32_t R) {
  return dtype == XL_C64 ? solve_ws_bytes<float>(B, K, R) : solve_ws_bytes<double>(B, K, R);
}

int xl_solve(int dtype, int method, int variant, const void* A, int64_t B, int32_t K,
             const void* S, int32_t R, const void* w0, const double* precond,
             int32_t precond_identity, int32_t T, double eps, void* X, int32_t* iterations,
             double* trace, void* iterates, int32_t* status, void* workspace,
             size_t ws_bytes, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (method != XL_JACPCG && method != XL_CG && method != XL_DIRECT) { set_error("unknown method %d", method); return XL_ERR_CONFIG; }
  if (variant != XL_TEXTBOOK && variant != XL_ALGORITHM) { set_error("unknown PCG variant %d", variant); return XL_ERR_CONFIG; }
  if (method != XL_DIRECT && T < 1) { set_error("iteration count T must be >= 1, got %d", T); return XL_ERR_CONFIG; }
  if (K < 1 || R < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (!S && R != K) { set_error("identity RHS needs R == K"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  SolveArgs a{method, variant, A, B, K, S, R, w0, precond, precond_identity, T, eps,
              X, iterations, trace, iterates, status, workspace, ws_bytes};
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == XL_C64 ? launch_solve<float>(a, st) : launch_solve<double>(a, st);
}

int xl_solve_stationary(int dtype, int method, const void* A, int64_t B, int32_t K,
                        const void* S, int32_t R, const void* w0, double omega, int32_t T,
                        double eps, void* X, int32_t* iterations, double* trace, void* iterates,
                        int32_t* status, void* workspace, size_t ws_bytes, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (method != XL_JOR && method != XL_GS) { set_error("unknown stationary method %d", method); return XL_ERR_CONFIG; }
  if (T < 1) { set_error("iteration count T must be >= 1, got %d", T); return XL_ERR_CONFIG; }
  if (method == XL_JOR && !(omega > 0)) { set_error("relaxation omega must be positive, got %g", omega); return XL_ERR_CONFIG; }
  if (K < 1 || R < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (!S && R != K) { set_error("identity RHS needs R == K"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  SolveArgs a{method, XL_TEXTBOOK, A, B, K, S, R, w0, nullptr, 0, T, eps,
              X, iterations, trace, iterates, status, workspace, ws_bytes};
  a.omega = omega;
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == XL_C64 ? launch_solve<float>(a, st) : launch_solve<double>(a, st);
}

// ---------------------------------------------------------------------------
// Fused precoder.  Workspace (SIMT path): A | X | solver ws (reused for the
// coupling matrix) | ||F||^2 partials | iterations.
// ---------------------------------------------------------------------------
static size_t simt_rzf_ws(int dtype, int64_t B, int M, int K) {
  size_t cs = csize(dtype), kk = (size_t)B * K * K * cs;
  size_t sws = xl_solve_workspace_bytes(dtype, B, K, K);
  if (sws < kk) sws = kk;
  const int tiles = gemm_tiles(M, K) > gemm_tiles(K, K) ? gemm_tiles(M, K) : gemm_tiles(K, K);
  return align_up(kk) + align_up(kk) + align_up(sws) +
         align_up((size_t)B * tiles * sizeof(double)) + align_up((size_t)B * 4);
}

// Large K: the general path runs its Gram / W products on the tensor cores
// (gemm_tc.cu).  Their split operands [Zh | Zl] take twice the bytes of H; they
// are kept for the whole batch (up to 32 GiB, i.e. 16 GiB of H) so the W
// products reuse them, else built per sub-batch for the Gram and again for W.
static int64_t tc_chunk_size(int dtype, int64_t B, int M, int K) {
  if (dtype == XL_C128) return B;
  const int64_t per = (int64_t)M * 4 * K * 4;  // split rows [Zh | Zl] per realization
  int64_t c = ((int64_t)32 << 30) / per;
  if (c < 1) c = 1;
  return c < B ? c : B;
}

// K = 128 complex64 with M % 64 == 0: the streaming Gram / W kernels
// (stream_tc.cu) need one split scale and one range flag per realization
// (below) and only the cuBLAS workspace the split-GEMM solver may still use.
static size_t stc_ws(int64_t, int) { return tc_cublas_ws_bytes(); }
// bytes of the tensor-core region that precedes the PCG buffers
static size_t tc_region(int dtype, int64_t B, int M, int K) {
  return stc_supported(dtype, M, K) ? stc_ws(B, K) : tc_gram_ws_bytes(dtype, tc_chunk_size(dtype, B, M, K), M, K);
}

static size_t general_ws(int dtype, int64_t B, int M, int K) {
  size_t w = simt_rzf_ws(dtype, B, M, K);
  if (lk_supported(dtype, M, K)) return w + align_up(lk_ws_bytes(B));
  if (tc_general_supported(dtype, M, K)) {
    if (stc_supported(dtype, M, K)) w += 2 * align_up((size_t)B * 4);  // sz[B], range flags[B]
    w += align_up(tc_region(dtype, B, M, K));
    if (dtype == XL_C64 && tc_pcg_supported(K)) w += align_up(tc_pcg_ws_bytes(B, K));
    if (dtype == XL_C128 && tc_pcg64_supported(K)) w += align_up(tc_pcg64_ws_bytes(B, K));
  }
  return w;
}

size_t xl_rzf_workspace_bytes(int dtype, int method, int64_t B, int32_t M, int32_t K) {
  if (fused_supported(dtype, method, M, K)) return fused_ws_bytes(dtype, method, B, M, K);
  return general_ws(dtype, B, M, K);
}

size_t xl_rzf_general_workspace_bytes(int dtype, int method, int64_t B, int32_t M, int32_t K) {
  (void)method;
  return general_ws(dtype, B, M, K);
}

// K = 256 complex64 Jac-PCG / CG (no telemetry): the batch in chunks whose
// kernels overlap across two streams -- the cluster solver of chunk i (a
// persistent grid of 4-CTA clusters on 132 of the 148 SMs, latency- and
// shared-memory-bound) runs while the Gram of chunk i + 1 and the beta / W /
// SINR of chunk i - 1 fill the remaining SMs and the solver's tail waves.
// XL_LK_PIPE=0: one chunk (the three kernels back to back).
static int lk_pipeline(int method, int variant, const void* H, int64_t B, int32_t M, double xi,
                       const double* xi_b, double power, int32_t T, double sigma2, void* W, void* F, double* beta,
                       double* gamma, double* sum_se, void* Xo, int32_t* status, void* A, void* GX, double* part,
                       void* tcws, cudaStream_t st) {
  constexpr int K = 256, NP = 8;  // part entries per realization (one per 32-column block)
  const LkScratch sc = lk_scratch(tcws, B);
  const size_t oH = (size_t)M * K * 8, oK = (size_t)K * K * 8;
  int64_t Bc = B;
  const char* pe = getenv("XL_LK_PIPE");
  if (!(pe && pe[0] == '0') && B >= 1024) Bc = B / 8 >= 512 ? (B + 7) / 8 : 512;
  const int64_t n = (B + Bc - 1) / Bc;
  auto gram = [&](int64_t b0, int64_t nb, cudaStream_t s) {
    return lk_gram((const char*)H + b0 * oH, nb, M, xi, xi_b ? xi_b + b0 : nullptr, (char*)A + b0 * oK, sc.sz + b0,
                   sc.rflag + b0, sc.zmax + b0, s);
  };
  auto solve = [&](int64_t b0, int64_t nb, cudaStream_t s) {
    return lk_solve(method, variant, (const char*)A + b0 * oK, nb, T, xi, xi_b ? xi_b + b0 : nullptr,
                    (char*)Xo + b0 * oK, (char*)GX + b0 * oK, part + b0 * NP, status + b0, sc.slots, s);
  };
  auto finish = [&](int64_t b0, int64_t nb, cudaStream_t s) {
    int e;
    if ((e = launch_beta_from_partials(nb, part + b0 * NP, NP, power, beta + b0, status + b0, s))) return e;
    if ((e = lk_apply((const char*)H + b0 * oH, (const char*)Xo + b0 * oK, beta + b0, nb, M, (char*)W + b0 * oH,
                      F ? (char*)F + b0 * oH : nullptr, sc.zmax + b0, lk_xmax((char*)GX + b0 * oK, nb), s)))
      return e;
    return lk_sinr((char*)GX + b0 * oK, beta + b0, nb, sigma2, gamma ? gamma + b0 * K : nullptr, sum_se + b0, s);
  };
  int e;
  if (n == 1) {
    if ((e = gram(0, B, st)) || (e = solve(0, B, st))) return e;
    return finish(0, B, st);
  }
  // a second stream and events per host thread and device (fork / join also inside graph capture)
  struct Side {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[2 * 8 + 2];
  };
  constexpr int MAX_DEV = 64;
  static thread_local Side side[MAX_DEV];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAX_DEV) { set_error("lk pipeline: device %d out of range", dev); return XL_ERR_UNSUPPORTED; }
  Side& sd = side[dev];
  if (sd.aux == nullptr) {
    if (cudaStreamCreateWithFlags(&sd.aux, cudaStreamNonBlocking) != cudaSuccess) return check_launch("lk aux stream");
    for (auto& x : sd.ev)
      if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) return check_launch("lk events");
  }
  cudaStream_t aux = sd.aux;
  cudaEvent_t *ev_g = sd.ev, *ev_p = sd.ev + 8, ev_fork = sd.ev[16], ev_join = sd.ev[17];
  if (cudaEventRecord(ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(aux, ev_fork, 0) != cudaSuccess)
    return check_launch("lk fork");
  if ((e = gram(0, Bc, st))) return e;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b0 = i * Bc, nb = B - b0 < Bc ? B - b0 : Bc;
    if (i > 0 && cudaStreamWaitEvent(st, ev_g[i], 0) != cudaSuccess) return check_launch("lk wait gram");
    if ((e = solve(b0, nb, st))) return e;
    if (cudaEventRecord(ev_p[i], st) != cudaSuccess) return check_launch("lk record solve");
    if (i + 1 < n) {
      const int64_t b1 = b0 + Bc, nb1 = B - b1 < Bc ? B - b1 : Bc;
      if ((e = gram(b1, nb1, aux))) return e;
      if (cudaEventRecord(ev_g[i + 1], aux) != cudaSuccess) return check_launch("lk record gram");
    }
    if (cudaStreamWaitEvent(aux, ev_p[i], 0) != cudaSuccess) return check_launch("lk wait solve");
    if ((e = finish(b0, nb, aux))) return e;
  }
  if (cudaEventRecord(ev_join, aux) != cudaSuccess || cudaStreamWaitEvent(st, ev_join, 0) != cudaSuccess)
    return check_launch("lk join");
  return XL_SUCCESS;
}

static void* g_dbg_gram = nullptr;
void xl_debug_set_gram_out(void* A) { g_dbg_gram = A; }
void xl_debug_lk_trace(void* buf) { lk_debug_trace(buf); }

// The general path over B realizations (workspace: simt_rzf_ws(B) + the
// tensor-core sub-batch buffers).
static int general_path(int dtype, int method, int variant, const void* H, int64_t B, int32_t M, int32_t K,
                         double xi, const double* xi_per_batch, double power, int32_t T, double sigma2, void* W,
                         void* F, double* beta, double* gamma, double* sum_se, void* X, int32_t* status,
                         void* workspace, cudaStream_t st, double* trace = nullptr,
                         int32_t* iterations = nullptr) {
  // solver telemetry (xl_rzf_traced) comes from the SIMT solver, which records it
  const bool telemetry = trace != nullptr || iterations != nullptr;
  const bool lkp = lk_supported(dtype, M, K);
  const bool tc = !lkp && tc_general_supported(dtype, M, K);
  const size_t cs = csize(dtype), kk = (size_t)B * K * K * cs;
  char* p = (char*)workspace;
  void* A = p; p += align_up(kk);
  void* Xw = p; p += align_up(kk);
  size_t sws = xl_solve_workspace_bytes(dtype, B, K, K);
  if (sws < kk) sws = kk;
  void* sw = p; p += align_up(sws);
  const int ptiles = gemm_tiles(M, K) > gemm_tiles(K, K) ? gemm_tiles(M, K) : gemm_tiles(K, K);
  double* part = (double*)p; p += align_up((size_t)B * ptiles * sizeof(double));
  int32_t* iters = (int32_t*)p; p += align_up((size_t)B * 4);
  const bool sc = tc && stc_supported(dtype, M, K);
  float* szb = nullptr;
  int* rflag = nullptr;
  if (sc) {
    szb = (float*)p; p += align_up((size_t)B * 4);
    rflag = (int*)p; p += align_up((size_t)B * 4);
  }
  void* tcws = p;  // gemm_tc.cu: cuBLAS workspace + split operands (+ the tensor-core PCG state)
  void* pcgws = tc ? (void*)(p + align_up(tc_region(dtype, B, M, K))) : nullptr;
  void* Xo = X ? X : Xw;
  const xl_stream_t stream = (xl_stream_t)st;
  int e;
  if (lkp && !telemetry && method != XL_DIRECT)
    return lk_pipeline(method, variant, H, B, M, xi, xi_per_batch, power, T, sigma2, W, F, beta, gamma, sum_se, Xo,
                       status, A, sw, part, tcws, st);
  const int64_t Bc = tc ? tc_chunk_size(dtype, B, M, K) : B;
  const int64_t oH = (int64_t)M * K * (int64_t)cs, oK = (int64_t)K * K * (int64_t)cs;
  if (lkp) {  // K = 256: upper-triangular tcgen05 tiles, A emitted from TMEM
    const LkScratch ls = lk_scratch(tcws, B);
    if ((e = lk_gram(H, B, M, xi, xi_per_batch, A, ls.sz, ls.rflag, ls.zmax, st))) return e;
  } else if (sc) {  // streaming tcgen05 Gram, A emitted from TMEM
    if ((e = stc_gram(H, B, M, K, xi, xi_per_batch, szb, A, rflag, st))) return e;
  } else if (tc) {
    for (int64_t b0 = 0; b0 < B; b0 += Bc) {
      const int64_t nb = B - b0 < Bc ? B - b0 : Bc;
      if ((e = tc_gram(dtype, (const char*)H + b0 * oH, nb, M, K, xi_per_batch ? xi_per_batch + b0 : nullptr, xi,
                       (char*)A + b0 * oK, tcws, st)))
        return e;
    }
  } else if ((e = xl_gram(dtype, H, B, M, K, xi, xi_per_batch, A, stream))) {
    return e;
  }
  // W = beta H X on the tensor cores, per sub-batch (the split rows are rebuilt:
  // the Gram sub-batches have overwritten them)
  auto tc_w = [&]() -> int {
    if (lkp) return lk_apply(H, Xo, beta, B, M, W, F, lk_scratch(tcws, B).zmax, nullptr, st);
    if (sc) return stc_apply(H, Xo, beta, szb, B, M, K, W, F, st);
    for (int64_t b0 = 0; b0 < B; b0 += Bc) {
      const int64_t nb = B - b0 < Bc ? B - b0 : Bc;
      if (int r = tc_apply(dtype, (const char*)H + b0 * oH, (const char*)Xo + b0 * oK, beta + b0, nb, M, K,
                           (char*)W + b0 * oH, F ? (char*)F + b0 * oH : nullptr, tcws, st, Bc < B))
        return r;
    }
    return XL_SUCCESS;
  };
  // K = 128 (complex64): the fused 2-CTA-cluster solver keeps the PCG state on
  // chip and also returns GX and the ||F||^2 partials (cluster_pcg.cu)
  const bool lks = !telemetry && lkp && method != XL_DIRECT;
  const bool cpc = !telemetry && tc && dtype == XL_C64 && method != XL_DIRECT && cpcg_supported(K);
  const bool tcp = !telemetry && tc && dtype == XL_C64 && method != XL_DIRECT && !cpc && tc_pcg_supported(K);
  const bool tcp64 = !telemetry && tc && dtype == XL_C128 && method != XL_DIRECT && tc_pcg64_supported(K);
  const int64_t sH = (int64_t)M * K, sK = (int64_t)K * K;
  const int np = gemm_tiles(K, K);
  void* GX = sw;  // the solver workspace is free again (>= B K K)
  if (lks) {
    if ((e = lk_solve(method, variant, A, B, T, xi, xi_per_batch, Xo, GX, part, status, lk_scratch(tcws, B).slots,
                      st)))
      return e;
  } else if (cpc) {
    if ((e = cpcg_solve(method, variant, A, B, K, T, xi, xi_per_batch, Xo, GX, part, status, st))) return e;
  } else if (tcp) {
    if ((e = tc_pcg(method, variant, A, B, K, T, Xo, status, tcws, pcgws, st))) return e;
  } else if (tcp64) {
    if ((e = tc_pcg64(method, variant, A, B, K, T, Xo, status, tcws, pcgws, st))) return e;
  } else if ((e = xl_solve(dtype, method, variant, A, B, K, nullptr, K, nullptr, nullptr, method == XL_CG,
                           T, -1.0, Xo, iterations ? iterations : iters, trace, nullptr, status, sw, sws,
                           stream))) {
    return e;
  }
  // Coupling and ||F||^2 from the K x K side: GX = (A - xi I) X,
  // ||F||_F^2 = Re tr(X^H GX) (precoder.py:64-70 with F = H X), beta, then
  // W = beta H X in one pass and B = H^H W = beta GX (metrics.py:35-44):
  // 8 K^3 instead of 8 M K^2 flops for the coupling, no separate F pass.
  if (dtype == XL_C64) {
    if (lks) {
      if ((e = launch_beta_from_partials(B, part, 8, power, beta, status, st))) return e;
    } else if (cpc) {
      if ((e = launch_beta_from_partials(B, part, 2, power, beta, status, st))) return e;
    } else if (tcp) {  // GX and the ||F||^2 partials on the tensor cores from the PCG state
      if ((e = tc_gx(xi_per_batch, xi, B, K, GX, part, tcws, pcgws, st))) return e;
      const int nt = (K + 31) / 32;
      if ((e = launch_beta_from_partials(B, part, nt * nt, power, beta, status, st))) return e;
    } else {
      if ((e = launch_cgemm<float>(false, EPI_GXF, A, sK, K, Xo, sK, K, GX, sK, K, B, K, K, K, xi_per_batch, xi, part, st))) return e;
      if ((e = launch_beta_from_partials(B, part, np, power, beta, status, st))) return e;
    }
    if (tc || lkp) {
      if ((e = tc_w())) return e;
    } else {
      if ((e = launch_cgemm<float>(false, EPI_BSCALE, H, sH, K, Xo, sK, K, W, sH, K, B, M, K, K, beta, 0, nullptr, st))) return e;
      if (F && (e = launch_cgemm<float>(false, EPI_STORE, H, sH, K, Xo, sK, K, F, sH, K, B, M, K, K, nullptr, 0, nullptr, st))) return e;
    }
    if (lks) return lk_sinr(GX, beta, B, sigma2, gamma, sum_se, st);
    return launch_sinr<float>(GX, B, K, sigma2, gamma, nullptr, sum_se, st, beta);
  }
  if (tcp64) {
    if ((e = tc_gx64(A, xi_per_batch, xi, B, K, GX, part, tcws, pcgws, st))) return e;
    const int nt = (K + 31) / 32;
    if ((e = launch_beta_from_partials(B, part, nt * nt, power, beta, status, st))) return e;
  } else {
    if ((e = launch_cgemm<double>(false, EPI_GXF, A, sK, K, Xo, sK, K, GX, sK, K, B, K, K, K, xi_per_batch, xi, part, st))) return e;
    if ((e = launch_beta_from_partials(B, part, np, power, beta, status, st))) return e;
  }
  if (tc) {
    if ((e = tc_w())) return e;
  } else {
    if ((e = launch_cgemm<double>(false, EPI_BSCALE, H, sH, K, Xo, sK, K, W, sH, K, B, M, K, K, beta, 0, nullptr, st))) return e;
    if (F && (e = launch_cgemm<double>(false, EPI_STORE, H, sH, K, Xo, sK, K, F, sH, K, B, M, K, K, nullptr, 0, nullptr, st))) return e;
  }
  return launch_sinr<double>(GX, B, K, sigma2, gamma, nullptr, sum_se, st, beta);
}

static int rzf_impl(bool allow_fused, int dtype, int method, int variant, const void* H, int64_t B,
                    int32_t M, int32_t K, double xi, const double* xi_per_batch, double power,
                    int32_t T, double sigma2, void* W, void* F, double* beta, double* gamma,
                    double* sum_se, void* X, int32_t* status, void* workspace, size_t ws_bytes,
                    xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (method != XL_JACPCG && method != XL_CG && method != XL_DIRECT) { set_error("unknown method %d", method); return XL_ERR_CONFIG; }
  if (variant != XL_TEXTBOOK && variant != XL_ALGORITHM) { set_error("unknown PCG variant %d", variant); return XL_ERR_CONFIG; }
  if (method != XL_DIRECT && T < 1) { set_error("iteration count T must be >= 1, got %d", T); return XL_ERR_CONFIG; }
  if (!xi_per_batch && !(xi > 0)) { set_error("regularization xi must be positive, got %g", xi); return XL_ERR_CONFIG; }
  if (!(sigma2 > 0)) { set_error("noise power must be positive, got %g", sigma2); return XL_ERR_CONFIG; }
  if (M < 1 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  cudaStream_t st = (cudaStream_t)stream;
  // complex64 K in {16, 32} with H in shared memory: one CTA per realization, mma.sync + SIMT solve
  if (allow_fused && fc64s_supported(dtype, method, M, K)) {
    if (cudaMemsetAsync(status, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return check_launch("memset");
    return fc64s_rzf(method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2, W, F, beta, gamma, sum_se, X,
                     status, st);
  }
  const bool fused = allow_fused && fused_supported(dtype, method, M, K);
  const size_t need = fused ? fused_ws_bytes(dtype, method, B, M, K) : general_ws(dtype, B, M, K);
  if (ws_bytes < need) { set_error("rzf: workspace too small"); return XL_ERR_WORKSPACE; }
  if (cudaMemsetAsync(status, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return check_launch("memset");

  if (fused)
    return launch_fused(dtype, method, variant, H, B, M, K, xi, xi_per_batch, power, T,
                        sigma2, W, F, beta, gamma, sum_se, X, status, workspace, ws_bytes,
                        g_dbg_gram, st);
  // complex128, K in {16, 32}: one fused DMMA kernel per realization (cfg1)
  if (allow_fused && fc128_supported(dtype, method, M, K))
    return fc128_rzf(method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2, W, F, beta, gamma, sum_se, X,
                     status, st);

  // ---- general path: Gram -> solve -> GX, beta -> W = beta H X -> SINR
  return general_path(dtype, method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2, W, F, beta,
                      gamma, sum_se, X, status, workspace, st);
}

int xl_rzf(int dtype, int method, int variant, const void* H, int64_t B, int32_t M,
           int32_t K, double xi, const double* xi_per_batch, double power, int32_t T,
           double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
           void* X, int32_t* status, void* workspace, size_t ws_bytes, xl_stream_t stream) {
  return rzf_impl(true, dtype, method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2,
                  W, F, beta, gamma, sum_se, X, status, workspace, ws_bytes, stream);
}

int xl_rzf_traced(int dtype, int method, int variant, const void* H, int64_t B, int32_t M, int32_t K,
                  double xi, const double* xi_per_batch, double power, int32_t T, double sigma2, void* W,
                  void* F, double* beta, double* gamma, double* sum_se, void* X, int32_t* iterations,
                  double* trace, int32_t* status, void* workspace, size_t ws_bytes, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (method != XL_JACPCG && method != XL_CG && method != XL_DIRECT) { set_error("unknown method %d", method); return XL_ERR_CONFIG; }
  if (variant != XL_TEXTBOOK && variant != XL_ALGORITHM) { set_error("unknown PCG variant %d", variant); return XL_ERR_CONFIG; }
  if (method != XL_DIRECT && T < 1) { set_error("iteration count T must be >= 1, got %d", T); return XL_ERR_CONFIG; }
  if (!xi_per_batch && !(xi > 0)) { set_error("regularization xi must be positive, got %g", xi); return XL_ERR_CONFIG; }
  if (!(sigma2 > 0)) { set_error("noise power must be positive, got %g", sigma2); return XL_ERR_CONFIG; }
  if (M < 1 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (!iterations) { set_error("rzf_traced: iterations is required"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  if (ws_bytes < general_ws(dtype, B, M, K)) { set_error("rzf_traced: workspace too small"); return XL_ERR_WORKSPACE; }
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return check_launch("memset");
  return general_path(dtype, method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2, W, F, beta, gamma,
                      sum_se, X, status, workspace, st, trace, iterations);
}

int xl_rzf_general(int dtype, int method, int variant, const void* H, int64_t B, int32_t M,
                   int32_t K, double xi, const double* xi_per_batch, double power, int32_t T,
                   double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
                   void* X, int32_t* status, void* workspace, size_t ws_bytes, xl_stream_t stream) {
  return rzf_impl(false, dtype, method, variant, H, B, M, K, xi, xi_per_batch, power, T, sigma2,
                  W, F, beta, gamma, sum_se, X, status, workspace, ws_bytes, stream);
}

size_t xl_apply_precoder_workspace_bytes(int dtype, int64_t B, int32_t M, int32_t K) {
  return align_up((size_t)B * K * K * csize(dtype)) + align_up((size_t)B * gemm_tiles(M, K) * sizeof(double));
}

int xl_apply_precoder(int dtype, const void* H, const void* X, int64_t B, int32_t M, int32_t K,
                      double power, double sigma2, void* W, void* F, double* beta, double* gamma,
                      double* sum_se, int32_t* status, void* workspace, size_t ws_bytes,
                      xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (!(sigma2 > 0)) { set_error("noise power must be positive, got %g", sigma2); return XL_ERR_CONFIG; }
  if (M < 1 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  if (ws_bytes < xl_apply_precoder_workspace_bytes(dtype, B, M, K)) { set_error("apply_precoder: workspace too small"); return XL_ERR_WORKSPACE; }
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return check_launch("memset");
  char* p = (char*)workspace;
  void* Bc = p; p += align_up((size_t)B * K * K * csize(dtype));
  double* part = (double*)p;
  return apply_precoder(dtype, H, X, B, M, K, power, sigma2, W, F, beta, gamma, sum_se, status,
                        part, Bc, st);
}

size_t xl_sinr_workspace_bytes(int dtype, int64_t B, int32_t K) {
  return align_up((size_t)B * K * K * csize(dtype));
}

int xl_sinr(int dtype, const void* H, const void* G, int64_t B, int32_t M, int32_t K,
            double sigma2, double* gamma, double* se, double* sum_se, void* workspace,
            size_t ws_bytes, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (!(sigma2 > 0)) { set_error("noise power must be positive, got %g", sigma2); return XL_ERR_CONFIG; }
  if (M < 1 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  if (ws_bytes < xl_sinr_workspace_bytes(dtype, B, K)) { set_error("sinr: workspace too small"); return XL_ERR_WORKSPACE; }
  cudaStream_t st = (cudaStream_t)stream;
  int64_t sH = (int64_t)M * K, sK = (int64_t)K * K;
  int e;
  if (dtype == XL_C64) {
    if ((e = launch_cgemm<float>(true, EPI_STORE, H, sH, K, G, sH, K, workspace, sK, K, B, K, K, M, nullptr, 0, nullptr, st))) return e;
    return launch_sinr<float>(workspace, B, K, sigma2, gamma, se, sum_se, st);
  }
  if ((e = launch_cgemm<double>(true, EPI_STORE, H, sH, K, G, sH, K, workspace, sK, K, B, K, K, M, nullptr, 0, nullptr, st))) return e;
  return launch_sinr<double>(workspace, B, K, sigma2, gamma, se, sum_se, st);
}

int xl_channel_generate(int dtype, uint64_t seed, int64_t first, int64_t B, int32_t S,
                        int32_t Ms, int32_t K, double p, const double* Rsqrt, double beta_bar,
                        double dmin, double dmax, void* H, int32_t* status, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (S < 1 || Ms < 2 || K < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (!(p > 0 && p <= 1)) { set_error("visibility probability must lie in (0, 1], got %g", p); return XL_ERR_CONFIG; }
  if (!(dmin > 0 && dmax >= dmin)) { set_error("bad distance range"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return check_launch("memset");
  return launch_channel(dtype, seed, first, B, S, Ms, K, p, Rsqrt, beta_bar, dmin, dmax, H, status, st);
}

int xl_se_partials(const double* sum_se, int64_t B, int64_t chunk, double* partials,
                   xl_stream_t stream) {
  if (chunk < 1 || B < 0) { set_error("bad chunk"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  return launch_se_partials(sum_se, B, chunk, partials, (cudaStream_t)stream);
}

int xl_se_combine(const double* partials, int64_t n_chunks, double* mean_sem, xl_stream_t stream) {
  if (n_chunks < 1) { set_error("xl_se_combine needs at least one chunk"); return XL_ERR_CONFIG; }
  return launch_se_combine(partials, n_chunks, mean_sem, (cudaStream_t)stream);
}

int xl_ber_errors(int dtype, const void* Bc, const int8_t* bits, const void* noise, int64_t B,
                  int32_t K, int32_t nsym, int64_t* errors, xl_stream_t stream) {
  if (int e = check_dtype(dtype)) return e;
  if (K < 1 || nsym < 1 || B < 0) { set_error("bad sizes"); return XL_ERR_CONFIG; }
  if (B == 0) return XL_SUCCESS;
  return launch_ber(dtype, Bc, bits, noise, B, K, nsym, errors, (cudaStream_t)stream);
}

}  // extern "C"
