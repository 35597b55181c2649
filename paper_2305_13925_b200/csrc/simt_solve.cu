// General batched HPD solvers on the SIMT pipes: textbook Jac-PCG, the
// paper's Algorithm 1, CG (linsolve.py:183-294) and Cholesky direct solve
// (linsolve.py:109-119), with the reference's full option set (any RHS, w0,
// preconditioner override, eps early stop, residual trace, iterates).
//
// One CTA per realization.  The K x R iterate state lives in an L2-resident
// workspace laid out column-major ([j][i], one RHS column contiguous) so that
// every per-column inner product is a coalesced warp reduction in a fixed
// order (bit-reproducible, no float atomics).  A*M products go through
// shared-memory tiles.  This is the general path; the fused tensor-core
// precoder kernel covers the identity-RHS / w0 = 0 / fixed-T hot case.
#include <math.h>

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {

constexpr int ST = 256;  // threads per solver CTA

// Re(conj(a) * b); the ONE inner-product kernel of every variant, so that
// Jac-PCG with C = I reproduces CG bit-for-bit (linsolve.py:218-219).
template <typename C> __device__ __forceinline__ auto dotc_re(C a, C b) { return a.x * b.x + a.y * b.y; }

// out[:, j] = A * in[:, j], j < Rc; A row-major K x K; in/out column-major.
// UPPER: only the strict upper triangle of A (Gauss-Seidel's Up, linsolve.py:139).
template <typename R, bool UPPER = false>
__device__ void cta_gemm(const cplx<R>* __restrict__ A, const cplx<R>* in, cplx<R>* out,
                         int K, int Rc, cplx<R> (*As)[33], cplx<R> (*Ms)[33]) {
  using C = cplx<R>;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  for (int i0 = 0; i0 < K; i0 += 32)
    for (int j0 = 0; j0 < Rc; j0 += 32) {
      C acc[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[a][c] = mk<R>(0, 0);
      for (int l0 = 0; l0 < K; l0 += 16) {
        __syncthreads();
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          int e = tid + p * ST, r = e / 16, l = e % 16;
          C va = mk<R>(0, 0), vm = mk<R>(0, 0);
          if (i0 + r < K && l0 + l < K && (!UPPER || l0 + l > i0 + r)) va = A[(int64_t)(i0 + r) * K + l0 + l];
          if (j0 + r < Rc && l0 + l < K) vm = in[(int64_t)(j0 + r) * K + l0 + l];
          As[l][r] = va;
          Ms[l][r] = vm;
        }
        __syncthreads();
#pragma unroll
        for (int l = 0; l < 16; ++l) {
          C a0 = As[l][tx], a1 = As[l][tx + 16], m0 = Ms[l][ty], m1 = Ms[l][ty + 16];
          cfma(acc[0][0], a0, m0); cfma(acc[0][1], a0, m1);
          cfma(acc[1][0], a1, m0); cfma(acc[1][1], a1, m1);
        }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          int i = i0 + tx + 16 * a, j = j0 + ty + 16 * c;
          if (i < K && j < Rc) out[(int64_t)j * K + i] = acc[a][c];
        }
    }
  __syncthreads();
}

template <typename R>
__device__ __forceinline__ cplx<R> rhs_at(const cplx<R>* S, int i, int j, int Rc) {
  if (!S) return mk<R>(i == j ? (R)1 : (R)0, (R)0);
  return S[(int64_t)i * Rc + j];
}

// trace = ||A X - S||_F^2 (un-normalised) via Q; fixed-order reduction.
template <typename R>
__device__ double residual_norm2(const cplx<R>* A, const cplx<R>* X, cplx<R>* Q,
                                 const cplx<R>* S, int K, int Rc, cplx<R> (*As)[33],
                                 cplx<R> (*Ms)[33], double* colpart) {
  cta_gemm<R>(A, X, Q, K, Rc, As, Ms);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < Rc; j += ST / 32) {
    double acc = 0.0;
    for (int i = lane; i < K; i += 32) {
      cplx<R> e = csub(Q[(int64_t)j * K + i], rhs_at<R>(S, i, j, Rc));
      acc += (double)cabs2(e);
    }
    acc = warp_sum(acc);
    if (lane == 0) colpart[j] = acc;
  }
  __syncthreads();
  __shared__ double tot;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < Rc; ++j) t += colpart[j];
    tot = t;
  }
  __syncthreads();
  return tot;
}

template <typename R>
__global__ void __launch_bounds__(ST, sizeof(R) == 4 ? 4 : 2)
pcg_kernel(SolveArgs a) {
  using C = cplx<R>;
  const int64_t b = blockIdx.x;
  const int K = a.K, Rc = a.R;
  const C* A = (const C*)a.A + b * (int64_t)K * K;
  const C* S = a.S ? (const C*)a.S + b * (int64_t)K * Rc : nullptr;
  const int64_t per = (int64_t)K * Rc;
  C* Xw = (C*)a.ws + b * 4 * per;
  C* Rw = Xw + per;
  C* Mw = Rw + per;
  C* Qw = Mw + per;

  __shared__ C As[16][33], Ms[16][33];
  extern __shared__ double dyn[];
  double* colpart = dyn;            // Rc
  R* rz = (R*)(colpart + Rc);       // Rc  (rz for textbook, rr for cg/algorithm)
  R* cdiag = rz + Rc;               // K
  __shared__ int any_active, not_hpd, zero_diag;
  __shared__ double snorm2;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool textbook = (a.method == XL_JACPCG && a.variant == XL_TEXTBOOK);
  const bool use_c = (a.method == XL_JACPCG);  // cg: C = I (division skipped: exact)
  const bool want_trace = a.trace != nullptr || a.eps >= 0.0;

  if (tid == 0) { any_active = 0; not_hpd = 0; zero_diag = 0; }
  __syncthreads();
  for (int i = tid; i < K; i += ST) {
    R c = (R)1;
    if (use_c && !a.precond_identity) c = a.precond ? (R)a.precond[b * K + i] : A[(int64_t)i * K + i].x;
    cdiag[i] = c;
    if (c == (R)0) zero_diag = 1;
  }
  // ||S||^2 (linsolve.py:84-85)
  for (int j = warp; j < Rc; j += ST / 32) {
    double acc = 0.0;
    for (int i = lane; i < K; i += 32) acc += (double)cabs2(rhs_at<R>(S, i, j, Rc));
    acc = warp_sum(acc);
    if (lane == 0) colpart[j] = acc;
  }
  __syncthreads();
  if (zero_diag) {  // linsolve.py:205-208
    if (tid == 0) { a.status[b] = XL_STATUS_SPLITTING; a.iterations[b] = 0; }
    return;
  }
  if (tid == 0) {
    double t = 0.0;
    for (int j = 0; j < Rc; ++j) t += colpart[j];
    snorm2 = t > 0.0 ? t : 1.0;
  }
  // X = w0 (or 0); Q = A X
  for (int64_t e = tid; e < per; e += ST) {
    int j = (int)(e / K), i = (int)(e % K);
    Xw[e] = a.w0 ? ((const C*)a.w0)[b * per + (int64_t)i * Rc + j] : mk<R>(0, 0);
  }
  __syncthreads();
  __shared__ double sh_tr0;
  if (a.w0) {
    double t = residual_norm2<R>(A, Xw, Qw, S, K, Rc, As, Ms, colpart);  // leaves A X in Q
    if (tid == 0) sh_tr0 = t;
  } else {
    for (int64_t e = tid; e < per; e += ST) Qw[e] = mk<R>(0, 0);
    if (tid == 0) { double t = 0.0; for (int j = 0; j < Rc; ++j) t += colpart[j]; sh_tr0 = t; }
  }
  __syncthreads();
  const double tr0 = sh_tr0;
  if (a.trace && tid == 0) a.trace[b * (a.T + 1)] = tr0 / snorm2;

  // r = S - A w (algorithm: divided by C); z; m; rz  (linsolve.py:224-229, 264-268)
  for (int j = warp; j < Rc; j += ST / 32) {
    R acc = 0;
    for (int i = lane; i < K; i += 32) {
      int64_t e = (int64_t)j * K + i;
      C r = csub(rhs_at<R>(S, i, j, Rc), Qw[e]);
      if (use_c && !textbook) { r.x = r.x / cdiag[i]; r.y = r.y / cdiag[i]; }
      C z = r;
      if (textbook) { z.x = r.x / cdiag[i]; z.y = r.y / cdiag[i]; }
      Rw[e] = r;
      Mw[e] = z;
      acc += dotc_re(r, z);
    }
    acc = warp_sum(acc);
    if (lane == 0) { rz[j] = acc; if (acc > 0) any_active = 1; }
  }
  __syncthreads();

  int it = 0;
  for (int t = 1; t <= a.T; ++t) {
    if (!any_active) break;                              // linsolve.py:273-274
    cta_gemm<R>(A, Mw, Qw, K, Rc, As, Ms);               // Pm = P @ m
    if (tid == 0) any_active = 0;
    __syncthreads();
    for (int j = warp; j < Rc; j += ST / 32) {
      const R rzj = rz[j];
      const bool act = rzj > (R)0;
      R curv = 0;
      for (int i = lane; i < K; i += 32) {
        int64_t e = (int64_t)j * K + i;
        C q = Qw[e];
        if (!textbook && use_c) { q.x = q.x / cdiag[i]; q.y = q.y / cdiag[i]; }
        curv += dotc_re(Mw[e], q);
      }
      curv = warp_sum(curv);
      if (curv <= (R)0 && act) not_hpd = 1;              // linsolve.py:277-279
      const R alpha = act ? rzj / (curv > (R)0 ? curv : (R)1) : (R)0;
      R acc = 0;
      for (int i = lane; i < K; i += 32) {
        int64_t e = (int64_t)j * K + i;
        C q = Qw[e];
        if (!textbook && use_c) { q.x = q.x / cdiag[i]; q.y = q.y / cdiag[i]; }
        C m = Mw[e], x = Xw[e], r = Rw[e];
        x.x = x.x + alpha * m.x; x.y = x.y + alpha * m.y;
        r.x = r.x - alpha * q.x; r.y = r.y - alpha * q.y;
        C z = r;
        if (textbook) { z.x = r.x / cdiag[i]; z.y = r.y / cdiag[i]; }
        acc += dotc_re(r, z);
        Xw[e] = x;
        Rw[e] = r;
      }
      acc = warp_sum(acc);
      const R beta = act ? acc / (act ? rzj : (R)1) : (R)0;
      for (int i = lane; i < K; i += 32) {
        int64_t e = (int64_t)j * K + i;
        C r = Rw[e], m = Mw[e];
        C z = r;
        if (textbook) { z.x = r.x / cdiag[i]; z.y = r.y / cdiag[i]; }
        m.x = z.x + beta * m.x; m.y = z.y + beta * m.y;
        Mw[e] = m;
      }
      if (lane == 0) { rz[j] = acc; if (acc > (R)0) any_active = 1; }
    }
    __syncthreads();
    if (not_hpd) { if (tid == 0) a.status[b] = XL_STATUS_NOT_HPD; break; }
    it = t;
    double trt = 0.0;
    if (want_trace) {
      trt = residual_norm2<R>(A, Xw, Qw, S, K, Rc, As, Ms, colpart) / snorm2;
      if (a.trace && tid == 0) a.trace[b * (a.T + 1) + t] = trt;
    }
    if (a.iterates) {
      C* dst = (C*)a.iterates + (b * a.T + (t - 1)) * per;
      for (int64_t e = tid; e < per; e += ST) {
        int j = (int)(e / K), i = (int)(e % K);
        dst[(int64_t)i * Rc + j] = Xw[e];
      }
    }
    if (a.eps >= 0.0 && sqrt(trt) <= a.eps) break;       // linsolve.py:292-293
    __syncthreads();
  }
  __syncthreads();
  C* Xo = (C*)a.X + b * per;
  for (int64_t e = tid; e < per; e += ST) {
    int i = (int)(e / Rc), j = (int)(e % Rc);
    Xo[e] = Xw[(int64_t)j * K + i];
  }
  if (tid == 0) {
    a.iterations[b] = it;
    if (a.trace)
      for (int t = it + 1; t <= a.T; ++t) a.trace[b * (a.T + 1) + t] = __longlong_as_double(0x7ff8000000000000ll);
  }
}

// Cholesky P = L L^H then P^{-1} S by two triangular sweeps (cho_solve).
template <typename R>
__global__ void __launch_bounds__(ST)
chol_kernel(SolveArgs a) {
  using C = cplx<R>;
  const int64_t b = blockIdx.x;
  const int K = a.K, Rc = a.R;
  const C* A = (const C*)a.A + b * (int64_t)K * K;
  const C* S = a.S ? (const C*)a.S + b * (int64_t)K * Rc : nullptr;
  const int64_t per = (int64_t)K * Rc;
  C* L = (C*)a.ws + b * ((int64_t)K * K + 2 * per);  // column-major L(i,j) = L[j*K+i]
  C* Y = L + (int64_t)K * K;                          // column-major K x Rc
  C* Q = Y + per;
  __shared__ C As[16][33], Ms[16][33];
  extern __shared__ double dyn[];
  double* colpart = dyn;
  __shared__ int fail;
  __shared__ R dk;
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;
  for (int64_t e = tid; e < (int64_t)K * K; e += ST) {
    int j = (int)(e / K), i = (int)(e % K);
    L[e] = (i >= j) ? A[(int64_t)i * K + j] : mk<R>(0, 0);
  }
  for (int k = 0; k < K; ++k) {
    __syncthreads();
    if (tid == 0) {
      R d = L[(int64_t)k * K + k].x;
      if (!(d > (R)0)) fail = 1;                       // zpotrf: ajj <= 0 or NaN
      d = sqrt(d);
      dk = d;
      L[(int64_t)k * K + k] = mk<R>(d, (R)0);
    }
    __syncthreads();
    if (fail) break;
    const R d = dk;
    for (int i = k + 1 + tid; i < K; i += ST) {
      C v = L[(int64_t)k * K + i];
      v.x = v.x / d; v.y = v.y / d;
      L[(int64_t)k * K + i] = v;
    }
    __syncthreads();
    const int n = K - k - 1;
    for (int64_t e = tid; e < (int64_t)n * n; e += ST) {
      int jj = (int)(e / n), ii = (int)(e % n);
      if (ii < jj) continue;
      int i = k + 1 + ii, j = k + 1 + jj;
      C lik = L[(int64_t)k * K + i], ljk = L[(int64_t)k * K + j];
      C v = L[(int64_t)j * K + i];
      // v -= lik * conj(ljk)
      v.x = v.x - (lik.x * ljk.x + lik.y * ljk.y);
      v.y = v.y - (lik.y * ljk.x - lik.x * ljk.y);
      L[(int64_t)j * K + i] = v;
    }
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) { a.status[b] = XL_STATUS_CHOLESKY; a.iterations[b] = 0; }
    return;
  }
  for (int64_t e = tid; e < per; e += ST) {
    int j = (int)(e / K), i = (int)(e % K);
    Y[e] = rhs_at<R>(S, i, j, Rc);
  }
  // forward: L y = s
  for (int k = 0; k < K; ++k) {
    __syncthreads();
    const R d = L[(int64_t)k * K + k].x;
    for (int j = tid; j < Rc; j += ST) {
      C v = Y[(int64_t)j * K + k];
      v.x = v.x / d; v.y = v.y / d;
      Y[(int64_t)j * K + k] = v;
    }
    __syncthreads();
    const int n = K - k - 1;
    for (int64_t e = tid; e < (int64_t)n * Rc; e += ST) {
      int j = (int)(e / n), i = k + 1 + (int)(e % n);
      C v = Y[(int64_t)j * K + i];
      C l = L[(int64_t)k * K + i], y = Y[(int64_t)j * K + k];
      v.x = v.x - (l.x * y.x - l.y * y.y);
      v.y = v.y - (l.x * y.y + l.y * y.x);
      Y[(int64_t)j * K + i] = v;
    }
  }
  // backward: L^H x = y
  for (int k = K - 1; k >= 0; --k) {
    __syncthreads();
    const R d = L[(int64_t)k * K + k].x;
    for (int j = tid; j < Rc; j += ST) {
      C v = Y[(int64_t)j * K + k];
      v.x = v.x / d; v.y = v.y / d;
      Y[(int64_t)j * K + k] = v;
    }
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)k * Rc; e += ST) {
      int j = (int)(e / k), i = (int)(e % k);
      C v = Y[(int64_t)j * K + i];
      C l = L[(int64_t)i * K + k], y = Y[(int64_t)j * K + k];  // conj(L(k,i)) * y
      v.x = v.x - (l.x * y.x + l.y * y.y);
      v.y = v.y - (l.x * y.y - l.y * y.x);
      Y[(int64_t)j * K + i] = v;
    }
  }
  __syncthreads();
  C* Xo = (C*)a.X + b * per;
  for (int64_t e = tid; e < per; e += ST) {
    int i = (int)(e / Rc), j = (int)(e % Rc);
    Xo[e] = Y[(int64_t)j * K + i];
  }
  if (a.trace) {
    // ||S||^2 then ||P x - S||^2 (linsolve.py:118)
    const int warp = tid >> 5, lane = tid & 31;
    for (int j = warp; j < Rc; j += ST / 32) {
      double acc = 0.0;
      for (int i = lane; i < K; i += 32) acc += (double)cabs2(rhs_at<R>(S, i, j, Rc));
      acc = warp_sum(acc);
      if (lane == 0) colpart[j] = acc;
    }
    __syncthreads();
    __shared__ double sn;
    if (tid == 0) { double t = 0; for (int j = 0; j < Rc; ++j) t += colpart[j]; sn = t > 0 ? t : 1.0; }
    __syncthreads();
    double tr = residual_norm2<R>(A, Y, Q, S, K, Rc, As, Ms, colpart);
    if (tid == 0) a.trace[b] = tr / sn;
  }
  if (tid == 0) a.iterations[b] = 0;
}

// numpy's complex division (Smith's scaling, multiply by the reciprocal), so a
// real divisor gives the same rounding as the reference's (s - P w) / d.
template <typename R>
__device__ __forceinline__ cplx<R> cdiv_np(cplx<R> a, cplx<R> d) {
  const R ar = fabs(d.x), ai = fabs(d.y);
  if (ar >= ai) {
    const R rat = d.y / d.x, scl = (R)1 / (d.x + d.y * rat);
    return mk<R>((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  const R rat = d.x / d.y, scl = (R)1 / (d.y + d.x * rat);
  return mk<R>((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// Stationary splittings, one CTA per realization (linsolve.py:128-176):
//   XL_JOR: w <- w + omega * (s - P w) / diag(P)                  (:154-176)
//   XL_GS : w <- (D + Lo)^{-1} (s - Up w), forward substitution    (:128-151)
// Zero diagonal -> SplittingError (_check_diag :120-125).  Trace, eps stop and
// iterates as in the Krylov kernel; no curvature checks (the reference has none).
template <typename R>
__global__ void __launch_bounds__(ST)
stationary_kernel(SolveArgs a, double omega) {
  using C = cplx<R>;
  const int64_t b = blockIdx.x;
  const int K = a.K, Rc = a.R;
  const C* A = (const C*)a.A + b * (int64_t)K * K;
  const C* S = a.S ? (const C*)a.S + b * (int64_t)K * Rc : nullptr;
  const int64_t per = (int64_t)K * Rc;
  C* Xw = (C*)a.ws + b * 4 * per;
  C* Qw = Xw + per;
  C* Rw = Qw + per;
  __shared__ C As[16][33], Ms[16][33];
  extern __shared__ double dyn[];
  double* colpart = dyn;
  __shared__ int zero_diag;
  __shared__ double snorm2, sh_tr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool gs = a.method == XL_GS;
  const bool want_trace = a.trace != nullptr || a.eps >= 0.0;
  if (tid == 0) zero_diag = 0;
  __syncthreads();
  for (int i = tid; i < K; i += ST) {
    const C d = A[(int64_t)i * K + i];
    if (d.x == (R)0 && d.y == (R)0) zero_diag = 1;
  }
  for (int j = warp; j < Rc; j += ST / 32) {  // ||S||^2 (linsolve.py:84-85)
    double acc = 0.0;
    for (int i = lane; i < K; i += 32) acc += (double)cabs2(rhs_at<R>(S, i, j, Rc));
    acc = warp_sum(acc);
    if (lane == 0) colpart[j] = acc;
  }
  __syncthreads();
  if (zero_diag) {
    if (tid == 0) { a.status[b] = XL_STATUS_SPLITTING; a.iterations[b] = 0; }
    return;
  }
  if (tid == 0) {
    double t = 0.0;
    for (int j = 0; j < Rc; ++j) t += colpart[j];
    snorm2 = t > 0.0 ? t : 1.0;
  }
  for (int64_t e = tid; e < per; e += ST) {
    const int j = (int)(e / K), i = (int)(e % K);
    Xw[e] = a.w0 ? ((const C*)a.w0)[b * per + (int64_t)i * Rc + j] : mk<R>(0, 0);
  }
  __syncthreads();
  {
    const double t0 = residual_norm2<R>(A, Xw, Qw, S, K, Rc, As, Ms, colpart);
    if (a.trace && tid == 0) a.trace[b * (a.T + 1)] = t0 / snorm2;
  }
  int it = 0;
  for (int t = 1; t <= a.T; ++t) {
    if (!gs) {
      cta_gemm<R>(A, Xw, Qw, K, Rc, As, Ms);  // P w
      for (int64_t e = tid; e < per; e += ST) {
        const int j = (int)(e / K), i = (int)(e % K);
        const C u = cdiv_np<R>(csub(rhs_at<R>(S, i, j, Rc), Qw[e]), A[(int64_t)i * K + i]);
        C x = Xw[e];
        x.x = x.x + (R)omega * u.x;
        x.y = x.y + (R)omega * u.y;
        Xw[e] = x;
      }
    } else {
      cta_gemm<R, true>(A, Xw, Qw, K, Rc, As, Ms);  // Up w
      for (int64_t e = tid; e < per; e += ST) {
        const int j = (int)(e / K), i = (int)(e % K);
        Rw[e] = csub(rhs_at<R>(S, i, j, Rc), Qw[e]);
      }
      __syncthreads();
      // (D + Lo) w = rhs: one warp per RHS column, lanes own rows l = lane + 32 m;
      // step i finalises w_i and eliminates it from the rows below.
      for (int j = warp; j < Rc; j += ST / 32) {
        C* rj = Rw + (int64_t)j * K;
        C* xj = Xw + (int64_t)j * K;
        for (int i = 0; i < K; ++i) {
          C wi = mk<R>(0, 0);
          if (lane == (i & 31)) {
            wi = cdiv_np<R>(rj[i], A[(int64_t)i * K + i]);
            xj[i] = wi;
          }
          wi.x = __shfl_sync(0xffffffffu, wi.x, i & 31);
          wi.y = __shfl_sync(0xffffffffu, wi.y, i & 31);
          for (int l = i + 1 + ((lane - (i + 1)) & 31); l < K; l += 32) {
            const C p = A[(int64_t)l * K + i];
            C v = rj[l];
            v.x = v.x - (p.x * wi.x - p.y * wi.y);
            v.y = v.y - (p.x * wi.y + p.y * wi.x);
            rj[l] = v;
          }
        }
      }
    }
    __syncthreads();
    it = t;
    double trt = 0.0;
    if (want_trace) {
      trt = residual_norm2<R>(A, Xw, Qw, S, K, Rc, As, Ms, colpart) / snorm2;
      if (a.trace && tid == 0) a.trace[b * (a.T + 1) + t] = trt;
    }
    if (a.iterates) {
      C* dst = (C*)a.iterates + (b * a.T + (t - 1)) * per;
      for (int64_t e = tid; e < per; e += ST) {
        const int j = (int)(e / K), i = (int)(e % K);
        dst[(int64_t)i * Rc + j] = Xw[e];
      }
    }
    if (tid == 0) sh_tr = trt;
    __syncthreads();
    if (a.eps >= 0.0 && sqrt(sh_tr) <= a.eps) break;  // linsolve.py:148-149, 173-174
    __syncthreads();
  }
  __syncthreads();
  C* Xo = (C*)a.X + b * per;
  for (int64_t e = tid; e < per; e += ST) {
    const int i = (int)(e / Rc), j = (int)(e % Rc);
    Xo[e] = Xw[(int64_t)j * K + i];
  }
  if (tid == 0) {
    a.iterations[b] = it;
    if (a.trace)
      for (int t = it + 1; t <= a.T; ++t) a.trace[b * (a.T + 1) + t] = __longlong_as_double(0x7ff8000000000000ll);
  }
}

template <typename R> size_t solve_ws_bytes(int64_t B, int K, int Rc) {
  size_t per = (size_t)K * Rc;
  size_t pcg = 4 * per;
  size_t chol = (size_t)K * K + 2 * per;
  return (size_t)B * (pcg > chol ? pcg : chol) * sizeof(cplx<R>);
}

template <typename R> int launch_solve(const SolveArgs& a, cudaStream_t st) {
  if (a.ws_bytes < solve_ws_bytes<R>(a.B, a.K, a.R)) {
    set_error("solve: workspace too small");
    return XL_ERR_WORKSPACE;
  }
  size_t dyn = (size_t)a.R * sizeof(double) + ((size_t)a.R + a.K) * sizeof(R) + 16;
  if (dyn > 48 * 1024) { set_error("solve: too many columns (R=%d)", a.R); return XL_ERR_UNSUPPORTED; }
  if (a.method == XL_DIRECT) chol_kernel<R><<<(unsigned)a.B, ST, dyn, st>>>(a);
  else if (a.method == XL_JOR || a.method == XL_GS) stationary_kernel<R><<<(unsigned)a.B, ST, dyn, st>>>(a, a.omega);
  else pcg_kernel<R><<<(unsigned)a.B, ST, dyn, st>>>(a);
  return check_launch(a.method == XL_DIRECT ? "chol" : a.method == XL_JOR || a.method == XL_GS ? "stationary" : "pcg");
}

template size_t solve_ws_bytes<float>(int64_t, int, int);
template size_t solve_ws_bytes<double>(int64_t, int, int);
template int launch_solve<float>(const SolveArgs&, cudaStream_t);
template int launch_solve<double>(const SolveArgs&, cudaStream_t);

}  // namespace xl
