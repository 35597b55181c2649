// Batched complex GEMM / Gram / precoder epilogue kernels on the SIMT pipes.
//
// This is the general path: any (M, K), complex64 (fp32 FMA) and complex128
// (fp64 FMA; on B200 the FP64 vector rate equals the DMMA rate, so SIMT fp64
// is the native c128 path).  The c64 hot shapes are served by the fused
// tcgen05 kernel in fused_tc.cu; this file is the fallback and the c128 path.
//
// Reference ops replaced: H^H H (precoder.py:59-60), F = H X (precoder.py:90),
// ||F||_F^2 / beta / G = beta F (precoder.py:64-70), B = H^H G and the SINR
// formula (metrics.py:35-58).
#include <stdio.h>

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {

// Tile: 32x32 complex outputs, 16-deep K chunks, 256 threads, 2x2 per thread.
constexpr int TB = 32, TK = 16, NT = 256;

// op(A)[i][l]: CONJ_A -> conj(A[l][i]) with A stored (k x m, lda);
//              else   -> A[i][l] with A stored (m x k, lda).
template <typename R, bool CONJ_A, int EPI>
__global__ void __launch_bounds__(NT)
cgemm_kernel(const cplx<R>* __restrict__ A, int64_t sA, int lda,
             const cplx<R>* __restrict__ Bm, int64_t sB, int ldb,
             cplx<R>* __restrict__ Cm, int64_t sC, int ldc,
             int m, int n, int k, const double* __restrict__ diag_add,
             double diag_scalar, double* __restrict__ partial) {
  using C = cplx<R>;
  __shared__ C As[TK][TB + 1];
  __shared__ C Bs[TK][TB + 1];
  const int64_t b = blockIdx.x;
  int ti, tj;
  if (EPI == EPI_GRAM) {  // lower-triangle tile index -> (ti, tj), ti >= tj
    int t = blockIdx.y;
    ti = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    const int ntj = (n + TB - 1) / TB;
    ti = blockIdx.y / ntj;
    tj = blockIdx.y % ntj;
  }
  const int i0 = ti * TB, j0 = tj * TB;
  const C* Ab = A + b * sA;
  const C* Bb = Bm + b * sB;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  C acc[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 2; ++c) acc[a][c] = mk<R>(0, 0);

  for (int l0 = 0; l0 < k; l0 += TK) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      int e = tid + p * NT;  // 0..511 over a TK x TB tile
      if (CONJ_A) {          // A stored (k x m): row l, col i -> coalesced along i
        int l = e / TB, i = e % TB;
        C v = mk<R>(0, 0);
        if (l0 + l < k && i0 + i < m) v = cconj(Ab[(int64_t)(l0 + l) * lda + i0 + i]);
        As[l][i] = v;
      } else {               // A stored (m x k): row i, col l -> coalesced along l
        int i = e / TK, l = e % TK;
        C v = mk<R>(0, 0);
        if (l0 + l < k && i0 + i < m) v = Ab[(int64_t)(i0 + i) * lda + l0 + l];
        As[l][i] = v;
      }
      {
        int l = e / TB, j = e % TB;
        C v = mk<R>(0, 0);
        if (l0 + l < k && j0 + j < n) v = Bb[(int64_t)(l0 + l) * ldb + j0 + j];
        Bs[l][j] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < TK; ++l) {
      C a0 = As[l][ty], a1 = As[l][ty + 16];
      C b0 = Bs[l][tx], b1 = Bs[l][tx + 16];
      cfma(acc[0][0], a0, b0); cfma(acc[0][1], a0, b1);
      cfma(acc[1][0], a1, b0); cfma(acc[1][1], a1, b1);
    }
    __syncthreads();
  }

  C* Cb = Cm + b * sC;
  double local = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      int i = i0 + ty + 16 * a, j = j0 + tx + 16 * c;
      if (i >= m || j >= n) continue;
      C v = acc[a][c];
      if (EPI == EPI_GRAM) {
        if (i > j) {
          Cb[(int64_t)i * ldc + j] = v;
          Cb[(int64_t)j * ldc + i] = cconj(v);
        } else if (i == j) {
          double xi = diag_add ? diag_add[b] : diag_scalar;
          Cb[(int64_t)i * ldc + i] = mk<R>((R)((double)v.x + xi), (R)0);
        }
      } else if (EPI == EPI_GXF) {  // (A - xi I) X and Re<X, (A - xi I) X>
        const double xi = diag_add ? diag_add[b] : diag_scalar;
        const C x = Bb[(int64_t)i * ldb + j];
        v.x = (R)((double)v.x - xi * (double)x.x);
        v.y = (R)((double)v.y - xi * (double)x.y);
        Cb[(int64_t)i * ldc + j] = v;
        local += (double)x.x * (double)v.x + (double)x.y * (double)v.y;
      } else if (EPI == EPI_BSCALE) {  // per-batch scale (beta)
        const R sc = (R)diag_add[b];
        Cb[(int64_t)i * ldc + j] = cscale(v, sc);
      } else {
        Cb[(int64_t)i * ldc + j] = v;
        if (EPI == EPI_FNORM) local += (double)cabs2(v);
      }
    }
  if (EPI == EPI_FNORM || EPI == EPI_GXF) {
    // fixed-order block reduction -> one partial per (b, tile)
    __shared__ double red[NT / 32];
    local = warp_sum(local);
    if ((tid & 31) == 0) red[tid >> 5] = local;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[w];
      partial[b * gridDim.y + blockIdx.y] = s;
    }
  }
}

template <typename R>
int launch_cgemm(bool conjA, int epi, const void* A, int64_t sA, int lda,
                 const void* Bm, int64_t sB, int ldb, void* Cm, int64_t sC,
                 int ldc, int64_t batch, int m, int n, int k,
                 const double* diag_add, double diag_scalar, double* partial,
                 cudaStream_t st) {
  using C = cplx<R>;
  int nti = (m + TB - 1) / TB, ntj = (n + TB - 1) / TB;
  int tiles = (epi == EPI_GRAM) ? nti * (nti + 1) / 2 : nti * ntj;
  if (tiles > 65535) { set_error("cgemm: too many tiles (%d)", tiles); return XL_ERR_UNSUPPORTED; }
  dim3 grid((unsigned)batch, tiles);
#define XL_GEMM_ARGS (const C*)A, sA, lda, (const C*)Bm, sB, ldb, (C*)Cm, sC, ldc, m, n, k, diag_add, diag_scalar, partial
  if (conjA) {
    if (epi == EPI_GRAM) cgemm_kernel<R, true, EPI_GRAM><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
    else if (epi == EPI_FNORM) cgemm_kernel<R, true, EPI_FNORM><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
    else cgemm_kernel<R, true, EPI_STORE><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
  } else {
    if (epi == EPI_FNORM) cgemm_kernel<R, false, EPI_FNORM><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
    else if (epi == EPI_GXF) cgemm_kernel<R, false, EPI_GXF><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
    else if (epi == EPI_BSCALE) cgemm_kernel<R, false, EPI_BSCALE><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
    else cgemm_kernel<R, false, EPI_STORE><<<grid, NT, 0, st>>>(XL_GEMM_ARGS);
  }
#undef XL_GEMM_ARGS
  return check_launch("cgemm");
}

int gemm_tiles(int m, int n) { return ((m + TB - 1) / TB) * ((n + TB - 1) / TB); }

template int launch_cgemm<float>(bool, int, const void*, int64_t, int, const void*, int64_t, int, void*, int64_t, int, int64_t, int, int, int, const double*, double, double*, cudaStream_t);
template int launch_cgemm<double>(bool, int, const void*, int64_t, int, const void*, int64_t, int, void*, int64_t, int, int64_t, int, int, int, const double*, double, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// beta = sqrt(power / ||F||^2) from per-tile partials (fixed order), then
// W = beta * F in place (optionally keeping F).  precoder.py:64-70.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void beta_scale_kernel(cplx<R>* __restrict__ W, cplx<R>* __restrict__ F,
                                  int64_t per, const double* __restrict__ partial,
                                  int nparts, double power, double* __restrict__ beta,
                                  int32_t* __restrict__ status) {
  const int64_t b = blockIdx.y;
  __shared__ double sbeta;
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int p = 0; p < nparts; ++p) tr += partial[b * nparts + p];
    double bt = 0.0;
    if (!(tr > 0.0)) {
      if (status && status[b] == XL_STATUS_OK) status[b] = XL_STATUS_DEGENERATE;
    } else {
      bt = sqrt(power / tr);
    }
    sbeta = bt;
    if (blockIdx.x == 0) beta[b] = bt;
  }
  __syncthreads();
  const R bt = (R)sbeta;
  cplx<R>* Wb = W + b * per;
  cplx<R>* Fb = F ? F + b * per : nullptr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per;
       e += (int64_t)gridDim.x * blockDim.x) {
    cplx<R> v = Wb[e];
    if (Fb) Fb[e] = v;
    Wb[e] = cscale(v, bt);
  }
}

// beta = sqrt(power / ||F||^2) only (||F||^2 from per-tile partials).
__global__ void beta_kernel(int64_t B, const double* __restrict__ partial, int nparts, double power,
                            double* __restrict__ beta, int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  double tr = 0.0;
  for (int p = 0; p < nparts; ++p) tr += partial[b * nparts + p];
  double bt = 0.0;
  if (!(tr > 0.0)) {
    if (status && status[b] == XL_STATUS_OK) status[b] = XL_STATUS_DEGENERATE;
  } else {
    bt = sqrt(power / tr);
  }
  beta[b] = bt;
}
int launch_beta_from_partials(int64_t B, const double* partial, int nparts, double power, double* beta,
                              int32_t* status, cudaStream_t st) {
  beta_kernel<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(B, partial, nparts, power, beta, status);
  return check_launch("beta");
}

template <typename R>
int launch_beta_scale(void* W, void* F, int64_t B, int64_t per, const double* partial,
                      int nparts, double power, double* beta, int32_t* status,
                      cudaStream_t st) {
  int gx = (int)((per + 1023) / 1024);
  if (gx > 64) gx = 64;
  if (B > 65535) { set_error("beta_scale: batch too large for one launch"); return XL_ERR_UNSUPPORTED; }
  beta_scale_kernel<R><<<dim3(gx, (unsigned)B), 256, 0, st>>>(
      (cplx<R>*)W, (cplx<R>*)F, per, partial, nparts, power, beta, status);
  return check_launch("beta_scale");
}
template int launch_beta_scale<float>(void*, void*, int64_t, int64_t, const double*, int, double, double*, int32_t*, cudaStream_t);
template int launch_beta_scale<double>(void*, void*, int64_t, int64_t, const double*, int, double, double*, int32_t*, cudaStream_t);

// ---------------------------------------------------------------------------
// SINR / SE from the coupling matrix B (K x K), metrics.py:47-58.
// One warp per user row; sum over users in fixed index order.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void sinr_kernel(const cplx<R>* __restrict__ Bc, int K, double sigma2,
                            double* __restrict__ gamma, double* __restrict__ se,
                            double* __restrict__ sum_se, const double* __restrict__ bscale) {
  const int64_t b = blockIdx.x;
  const double s2 = bscale ? bscale[b] * bscale[b] : 1.0;  // B = beta * Bc
  extern __shared__ double sse[];
  const cplx<R>* Bb = Bc + b * (int64_t)K * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < K; k += nw) {
    double tot = 0.0;
    for (int j = lane; j < K; j += 32) tot += (double)cabs2(Bb[(int64_t)k * K + j]);
    tot = warp_sum(tot) * s2;
    double sig = (double)cabs2(Bb[(int64_t)k * K + k]) * s2;
    double g = sig / ((tot - sig) + sigma2);
    double s = log2(1.0 + g);
    if (lane == 0) {
      if (gamma) gamma[b * K + k] = g;
      if (se) se[b * K + k] = s;
      sse[k] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < K; ++k) t += sse[k];
    sum_se[b] = t;
  }
}

template <typename R>
int launch_sinr(const void* Bc, int64_t B, int K, double sigma2, double* gamma,
                double* se, double* sum_se, cudaStream_t st, const double* bscale) {
  sinr_kernel<R><<<(unsigned)B, 256, K * sizeof(double), st>>>(
      (const cplx<R>*)Bc, K, sigma2, gamma, se, sum_se, bscale);
  return check_launch("sinr");
}
template int launch_sinr<float>(const void*, int64_t, int, double, double*, double*, double*, cudaStream_t, const double*);
template int launch_sinr<double>(const void*, int64_t, int, double, double*, double*, double*, cudaStream_t, const double*);

// ---------------------------------------------------------------------------
// Ergodic-SE partials {sum, sum of squares, n} per chunk (metrics.py:61-68).
// ---------------------------------------------------------------------------
__global__ void se_partials_kernel(const double* __restrict__ s, int64_t B, int64_t chunk,
                                   double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const int64_t lo = c * chunk, hi = min(B, lo + chunk);
  __shared__ double r1[256], r2[256];
  double a = 0.0, q = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) { a += s[i]; q += s[i] * s[i]; }
  r1[threadIdx.x] = a; r2[threadIdx.x] = q;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) { r1[threadIdx.x] += r1[threadIdx.x + w]; r2[threadIdx.x] += r2[threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[3 * c] = r1[0]; out[3 * c + 1] = r2[0]; out[3 * c + 2] = (double)(hi - lo); }
}

// {mean, SEM (ddof = 1)} from ordered chunk partials, summed in chunk order by
// one thread (the few partials of a step; one launch instead of a dozen
// elementwise ones inside a replayed step)
__global__ void se_combine_kernel(const double* __restrict__ parts, int64_t nc, double* __restrict__ out) {
  double s = 0.0, q = 0.0, n = 0.0;
  for (int64_t c = 0; c < nc; ++c) {
    s += parts[3 * c];
    q += parts[3 * c + 1];
    n += parts[3 * c + 2];
  }
  const double mean = s / n;
  const double var = fmax(q - n * mean * mean, 0.0) / fmax(n - 1.0, 1.0);
  out[0] = mean;
  out[1] = n > 1.0 ? sqrt(var / n) : 0.0;
}

int launch_se_combine(const double* parts, int64_t nc, double* out, cudaStream_t st) {
  se_combine_kernel<<<1, 1, 0, st>>>(parts, nc, out);
  return check_launch("se_combine");
}

int launch_se_partials(const double* s, int64_t B, int64_t chunk, double* out, cudaStream_t st) {
  int64_t nc = (B + chunk - 1) / chunk;
  se_partials_kernel<<<(unsigned)nc, 256, 0, st>>>(s, B, chunk, out);
  return check_launch("se_partials");
}

}  // namespace xl
