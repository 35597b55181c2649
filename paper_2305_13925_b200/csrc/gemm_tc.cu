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

#include "xl_common.cuh"
#include "simt_kernels.cuh"

namespace xl {

namespace {

constexpr size_t CUBLAS_WS = 32u << 20;  // cuBLAS workspace carved from the caller's

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// One cuBLAS handle per (host thread, device): set stream / workspace calls on
// a handle are not safe against another thread using it concurrently.
cublasHandle_t handle_for_device() {
  thread_local cublasHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!handles[dev] && cublasCreate(&handles[dev]) != CUBLAS_STATUS_SUCCESS) {
    handles[dev] = nullptr;
    return nullptr;
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
// diagonal.  Exactly Hermitian by construction (real diagonal).  One CTA per 32 x 32
// tile of A: the 64 x 64 blocks of U and of U^T it needs are staged through shared
// memory with coalesced row reads; A is written row by row.
constexpr int XT = 32;
__global__ void __launch_bounds__(256) gram_extract_kernel(const float* __restrict__ U, float2* __restrict__ A,
                                                           int K, const double* __restrict__ xi_b, double xi) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const int i0 = blockIdx.z * XT, j0 = blockIdx.y * XT;
  const float* u = U + b * (int64_t)n2 * n2;
  __shared__ float t1[2 * XT][2 * XT + 1], t2[2 * XT][2 * XT + 1];  // U[2i0.., 2j0..], U[2j0.., 2i0..]
  for (int e = threadIdx.x; e < 4 * XT * XT; e += blockDim.x) {
    const int rr = e / (2 * XT), cc = e % (2 * XT);
    const int r1 = 2 * i0 + rr, c1 = 2 * j0 + cc, r2 = 2 * j0 + rr, c2 = 2 * i0 + cc;
    t1[rr][cc] = (r1 < n2 && c1 < n2) ? u[(int64_t)r1 * n2 + c1] : 0.0f;
    t2[rr][cc] = (r2 < n2 && c2 < n2) ? u[(int64_t)r2 * n2 + c2] : 0.0f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int ti = e / XT, tj = e % XT, i = i0 + ti, j = j0 + tj;
    if (i >= K || j >= K) continue;
    auto g = [&](int dr, int dc) { return 0.5f * (t1[2 * ti + dr][2 * tj + dc] + t2[2 * tj + dc][2 * ti + dr]); };
    float re = g(0, 0) + g(1, 1);
    float im = g(0, 1) - g(1, 0);
    if (i == j) {
      re = (float)((double)re + (xi_b ? xi_b[b] : xi));
      im = 0.0f;
    }
    A[b * (int64_t)K * K + (int64_t)i * K + j] = make_float2(re, im);
  }
}

// beta X (K x K complex) -> the split real embedding as the GEMM's A operands,
// column-major n2 x n2 views of row-major Xe (i.e. Xe^T):
//   E1 (n2 x 2 n2) = [Xeh^T | Xeh^T]  (pairs with S's [Zh ; Zl] rows)
//   E2 (n2 x n2)   = Xel^T            (pairs with Zh)
// Xe[2i][2j] = xr, Xe[2i][2j+1] = xi, Xe[2i+1][2j] = -xi, Xe[2i+1][2j+1] = xr.
__global__ void embed_x_kernel(const float2* __restrict__ X, const double* __restrict__ beta, float* __restrict__ E1,
                               float* __restrict__ E2, int K) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const float sc = (float)beta[b];
  float* e1 = E1 + b * (int64_t)n2 * 2 * n2;
  float* e2 = E2 + b * (int64_t)n2 * n2;
  const float2* xb = X + b * (int64_t)K * K;
  for (int r = blockIdx.y; r < n2; r += gridDim.y) {  // Xe row r: column r of the col-major view
    const float2* xrow = xb + (int64_t)(r >> 1) * K;
    for (int c = threadIdx.x; c < n2; c += blockDim.x) {
      const float2 x = xrow[c >> 1];
      const float xr = x.x * sc, xi = x.y * sc;
      const float v = (r & 1) == 0 ? ((c & 1) == 0 ? xr : xi) : ((c & 1) == 0 ? -xi : xr);
      const float h = tf32_rn(v);
      e1[(int64_t)r * n2 + c] = h;
      e1[(int64_t)(n2 + r) * n2 + c] = h;
      e2[(int64_t)r * n2 + c] = v - h;
    }
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




// ---------------------------------------------------------------------------
// Jac-PCG / CG on the real embedding for the rzf path at large K (identity
// right-hand sides, w0 = 0, fixed T): the K complex columns are K real columns
// of length n2 = 2K (column j = the complex column interleaved re/im, so the
// column-major real view IS the column-major complex state), A'' the real
// embedding of the Hermitian A (column 2j = A[:, j], column 2j+1 = i A[:, j]).
// Each iteration: Q = A'' P as two 3xTF32 GEMMs (E1 = [A''h | A''h] against the
// split P rows [Ph ; Pl], plus E2 = A''l against Ph), then one CTA per
// realization updates X, R, P with the per-column scalars of linsolve.py:217-294
// (textbook: z = r / c; Algorithm 1: r and Pm pre-divided by C; CG: C = I).
// Real inner products of the embedded columns are the complex Re(a^H b).
// ---------------------------------------------------------------------------

struct PcgState {
  float* E1;  // n2 x 2 n2 (col-major) per realization
  float* E2;  // n2 x n2
  float* SP;  // 2 n2 x K: [Ph ; Pl] per column
  float* Q;   // n2 x K
  float* P;   // n2 x K
  float* X;   // n2 x K
  float* R;   // n2 x K
  float* C;   // n2: preconditioner diagonal per real component (c_i twice)
  float* rz;  // K
};

__device__ __forceinline__ float warp_sum_f(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// build E1 / E2 from A (K x K complex row-major, Hermitian), C, and the initial state
__global__ void pcg_init_kernel(const float2* __restrict__ A, PcgState s, int K, int method, int variant,
                                int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const float2* a = A + b * (int64_t)K * K;
  float* e1 = s.E1 + b * (int64_t)n2 * 2 * n2;
  float* e2 = s.E2 + b * (int64_t)n2 * n2;
  float* c = s.C + b * (int64_t)n2;
  const bool use_c = method == XL_JACPCG;
  const bool textbook = use_c && variant == XL_TEXTBOOK;
  __shared__ int zero_diag;
  if (threadIdx.x == 0) zero_diag = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const float d = use_c ? a[(int64_t)i * K + i].x : 1.0f;
    if (d == 0.0f) zero_diag = 1;
    c[2 * i] = d;
    c[2 * i + 1] = d;
  }
  // A''(r, col): col 2j = A[:, j] (re/im interleaved), col 2j+1 = i A[:, j].  A is
  // Hermitian, so column j is conj(row j): read row j contiguously.
  for (int col = 0; col < n2; ++col) {
    const int j = col >> 1;
    const float2* arow = a + (int64_t)j * K;
    for (int r = threadIdx.x; r < n2; r += blockDim.x) {
      const float2 aji = arow[r >> 1];  // A_ij = conj(A_ji)
      const float re = aji.x, im = -aji.y;
      const float v = (col & 1) == 0 ? ((r & 1) == 0 ? re : im) : ((r & 1) == 0 ? -im : re);
      const float h = tf32_rn(v);
      e1[(int64_t)col * n2 + r] = h;
      e1[(int64_t)(n2 + col) * n2 + r] = h;
      e2[(int64_t)col * n2 + r] = v - h;
    }
  }
  __syncthreads();
  if (zero_diag) {
    if (threadIdx.x == 0) status[b] = XL_STATUS_SPLITTING;
  }
  // r = S - A w = I (Algorithm 1: C^-1 I), z, m = z, x = 0, rz (linsolve.py:224-229, 264-268)
  const int64_t per = (int64_t)n2 * K;
  float* P = s.P + b * per;
  float* X = s.X + b * per;
  float* R = s.R + b * per;
  float* SP = s.SP + b * 2 * per;
  for (int64_t e = threadIdx.x; e < per; e += blockDim.x) {
    const int j = (int)(e / n2), r = (int)(e % n2);
    const float ci = c[r];
    const bool one = r == 2 * j;
    const float rv = one ? ((use_c && !textbook) ? 1.0f / ci : 1.0f) : 0.0f;
    const float zv = textbook ? rv / ci : rv;
    R[e] = rv;
    X[e] = 0.0f;
    P[e] = zv;
    const float h = tf32_rn(zv);
    SP[(int64_t)j * 2 * n2 + r] = h;
    SP[(int64_t)j * 2 * n2 + n2 + r] = zv - h;
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const float ci = c[2 * j];
    s.rz[b * K + j] = textbook ? 1.0f / ci : ((use_c) ? (1.0f / ci) * (1.0f / ci) : 1.0f);
  }
}

// one PCG step after Q = A'' P (linsolve.py:275-288): one warp per column, the
// column's q, p, x, r held in registers (float4 per lane, n2 <= 512) so each is
// read and written once
constexpr int PCG_V = 4;  // float4 per lane and vector: n2 <= 32 * 4 * PCG_V
__global__ void pcg_update_kernel(PcgState s, int K, int method, int variant, int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K, nq = n2 / 4;
  const int64_t per = (int64_t)n2 * K;
  const bool use_c = method == XL_JACPCG;
  const bool textbook = use_c && variant == XL_TEXTBOOK;
  const float4* c4 = reinterpret_cast<const float4*>(s.C + b * (int64_t)n2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ int not_hpd;
  if (threadIdx.x == 0) not_hpd = 0;
  __syncthreads();
  for (int j = warp; j < K; j += nw) {
    const int64_t o = b * per + (int64_t)j * n2;
    const float4* q4 = reinterpret_cast<const float4*>(s.Q + o);
    float4* p4 = reinterpret_cast<float4*>(s.P + o);
    float4* x4 = reinterpret_cast<float4*>(s.X + o);
    float4* r4 = reinterpret_cast<float4*>(s.R + o);
    float4* sp4 = reinterpret_cast<float4*>(s.SP + b * 2 * per + (int64_t)j * 2 * n2);
    const float rzj = s.rz[b * K + j];
    const bool act = rzj > 0.0f;
    float4 qv[PCG_V], pv[PCG_V], cv[PCG_V];
    float curv = 0.0f;
#pragma unroll
    for (int t = 0; t < PCG_V; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        qv[t] = q4[i];
        pv[t] = p4[i];
        cv[t] = use_c ? c4[i] : make_float4(1.f, 1.f, 1.f, 1.f);
        if (use_c && !textbook) {
          qv[t].x = qv[t].x / cv[t].x; qv[t].y = qv[t].y / cv[t].y;
          qv[t].z = qv[t].z / cv[t].z; qv[t].w = qv[t].w / cv[t].w;
        }
        curv += pv[t].x * qv[t].x + pv[t].y * qv[t].y + pv[t].z * qv[t].z + pv[t].w * qv[t].w;
      }
    }
    curv = warp_sum_f(curv);
    if (curv <= 0.0f && act && lane == 0) not_hpd = 1;
    const float al = act ? rzj / (curv > 0.0f ? curv : 1.0f) : 0.0f;
    float acc = 0.0f;
    float4 rv[PCG_V];
#pragma unroll
    for (int t = 0; t < PCG_V; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        float4 xv = x4[i];
        rv[t] = r4[i];
        xv.x += al * pv[t].x; xv.y += al * pv[t].y; xv.z += al * pv[t].z; xv.w += al * pv[t].w;
        rv[t].x -= al * qv[t].x; rv[t].y -= al * qv[t].y; rv[t].z -= al * qv[t].z; rv[t].w -= al * qv[t].w;
        x4[i] = xv;
        r4[i] = rv[t];
        if (textbook)
          acc += rv[t].x * (rv[t].x / cv[t].x) + rv[t].y * (rv[t].y / cv[t].y) + rv[t].z * (rv[t].z / cv[t].z) +
                 rv[t].w * (rv[t].w / cv[t].w);
        else
          acc += rv[t].x * rv[t].x + rv[t].y * rv[t].y + rv[t].z * rv[t].z + rv[t].w * rv[t].w;
      }
    }
    acc = warp_sum_f(acc);
    const float be = act ? acc / rzj : 0.0f;
#pragma unroll
    for (int t = 0; t < PCG_V; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        float4 m;
        m.x = (textbook ? rv[t].x / cv[t].x : rv[t].x) + be * pv[t].x;
        m.y = (textbook ? rv[t].y / cv[t].y : rv[t].y) + be * pv[t].y;
        m.z = (textbook ? rv[t].z / cv[t].z : rv[t].z) + be * pv[t].z;
        m.w = (textbook ? rv[t].w / cv[t].w : rv[t].w) + be * pv[t].w;
        p4[i] = m;
        const float4 h = make_float4(tf32_rn(m.x), tf32_rn(m.y), tf32_rn(m.z), tf32_rn(m.w));
        sp4[i] = h;
        sp4[nq + i] = make_float4(m.x - h.x, m.y - h.y, m.z - h.z, m.w - h.w);
      }
    }
    if (lane == 0) s.rz[b * K + j] = acc;
  }
  __syncthreads();
  if (not_hpd && threadIdx.x == 0 && status[b] == 0) status[b] = XL_STATUS_NOT_HPD;
}

// column-major embedded X (n2 x K) -> row-major complex X (K x K): 32 x 32 tiles
// through shared memory (coalesced on both sides)
__global__ void __launch_bounds__(256) pcg_store_x_kernel(const float* __restrict__ Xs, float2* __restrict__ X,
                                                          int K) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const int i0 = blockIdx.z * XT, j0 = blockIdx.y * XT;
  __shared__ float2 t[XT][XT + 1];  // [j][i]
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int tj = e / XT, ti = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) {
      const float* col = Xs + b * (int64_t)n2 * K + (int64_t)j * n2;
      t[tj][ti] = make_float2(col[2 * i], col[2 * i + 1]);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int ti = e / XT, tj = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) X[b * (int64_t)K * K + (int64_t)i * K + j] = t[tj][ti];
  }
}

PcgState pcg_state(char* p, int64_t B, int K) {
  const size_t n2 = 2 * (size_t)K;
  PcgState s;
  s.E1 = (float*)p; p += align_up((size_t)B * n2 * 2 * n2 * 4);
  s.E2 = (float*)p; p += align_up((size_t)B * n2 * n2 * 4);
  s.SP = (float*)p; p += align_up((size_t)B * 2 * n2 * K * 4);
  s.Q = (float*)p; p += align_up((size_t)B * n2 * K * 4);
  s.P = (float*)p; p += align_up((size_t)B * n2 * K * 4);
  s.X = (float*)p; p += align_up((size_t)B * n2 * K * 4);
  s.R = (float*)p; p += align_up((size_t)B * n2 * K * 4);
  s.C = (float*)p; p += align_up((size_t)B * n2 * 4);
  s.rz = (float*)p;
  return s;
}

// [Xh ; Xl] split of the embedded X state (for the GX product)
__global__ void split_x_kernel(PcgState s, int K) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const int64_t per = (int64_t)n2 * K;
  for (int64_t e = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.y * blockDim.x) {
    const int j = (int)(e / n2), r = (int)(e % n2);
    const float v = s.X[b * per + e];
    const float h = tf32_rn(v);
    s.SP[b * 2 * per + (int64_t)j * 2 * n2 + r] = h;
    s.SP[b * 2 * per + (int64_t)j * 2 * n2 + n2 + r] = v - h;
  }
}

// GX = A'' X - xi X -> complex row-major K x K, and Re tr(X^H GX) partials: one per
// 32 x 32 tile (fixed-order sums, combined by the beta kernel in tile order)
__global__ void __launch_bounds__(256) gx_finish_kernel(PcgState s, int K, const double* __restrict__ xi_b, double xi,
                                                        float2* __restrict__ GX, double* __restrict__ part) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const int64_t per = (int64_t)n2 * K;
  const int i0 = blockIdx.z * XT, j0 = blockIdx.y * XT;
  const double x0 = xi_b ? xi_b[b] : xi;
  __shared__ float2 t[XT][XT + 1];  // [j][i]
  double local = 0.0;
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int tj = e / XT, ti = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) {
      const int64_t o = b * per + (int64_t)j * n2 + 2 * i;
      const float xr = s.X[o], xim = s.X[o + 1];
      const float gr = (float)((double)s.Q[o] - x0 * (double)xr);
      const float gi = (float)((double)s.Q[o + 1] - x0 * (double)xim);
      t[tj][ti] = make_float2(gr, gi);
      local += (double)xr * (double)gr + (double)xim * (double)gi;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int ti = e / XT, tj = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) GX[b * (int64_t)K * K + (int64_t)i * K + j] = t[tj][ti];
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tt = 0.0;
    for (int w = 0; w < 8; ++w) tt += red[w];
    part[b * gridDim.y * gridDim.z + blockIdx.z * gridDim.y + blockIdx.y] = tt;
  }
}


// ---------------------------------------------------------------------------
// complex128: the same recurrences with ZGEMM (FP64 tensor cores) for Q = A P
// directly on the complex state (no split: DMMA products are exact fp64).  The
// state is the column-major complex K x K matrix (column j = RHS j), read as
// real n2-vectors by the update kernel.
// ---------------------------------------------------------------------------
struct PcgState64 {
  double* Q;
  double* P;
  double* X;
  double* R;
  double* C;
  double* rz;
};

PcgState64 pcg_state64(char* p, int64_t B, int K) {
  const size_t n2 = 2 * (size_t)K;
  PcgState64 s;
  s.Q = (double*)p; p += align_up((size_t)B * n2 * K * 8);
  s.P = (double*)p; p += align_up((size_t)B * n2 * K * 8);
  s.X = (double*)p; p += align_up((size_t)B * n2 * K * 8);
  s.R = (double*)p; p += align_up((size_t)B * n2 * K * 8);
  s.C = (double*)p; p += align_up((size_t)B * n2 * 8);
  s.rz = (double*)p;
  return s;
}

__global__ void pcg_init64_kernel(const double2* __restrict__ A, PcgState64 s, int K, int method, int variant,
                                  int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K;
  const double2* a = A + b * (int64_t)K * K;
  double* c = s.C + b * (int64_t)n2;
  const bool use_c = method == XL_JACPCG;
  const bool textbook = use_c && variant == XL_TEXTBOOK;
  __shared__ int zero_diag;
  if (threadIdx.x == 0) zero_diag = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const double d = use_c ? a[(int64_t)i * K + i].x : 1.0;
    if (d == 0.0) zero_diag = 1;
    c[2 * i] = d;
    c[2 * i + 1] = d;
  }
  __syncthreads();
  if (zero_diag && threadIdx.x == 0) status[b] = XL_STATUS_SPLITTING;
  const int64_t per = (int64_t)n2 * K;
  for (int64_t e = threadIdx.x; e < per; e += blockDim.x) {
    const int j = (int)(e / n2), r = (int)(e % n2);
    const double ci = c[r];
    const double rv = r == 2 * j ? ((use_c && !textbook) ? 1.0 / ci : 1.0) : 0.0;
    s.R[b * per + e] = rv;
    s.X[b * per + e] = 0.0;
    s.P[b * per + e] = textbook ? rv / ci : rv;
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double ci = c[2 * j];
    s.rz[b * K + j] = textbook ? 1.0 / ci : (use_c ? (1.0 / ci) * (1.0 / ci) : 1.0);
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int PCG_V64 = 8;  // double2 per lane and vector: n2 <= 32 * 2 * PCG_V64
__global__ void __launch_bounds__(256) pcg_update64_kernel(PcgState64 s, int K, int method, int variant,
                                                           int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x;
  const int n2 = 2 * K, nq = n2 / 2;
  const int64_t per = (int64_t)n2 * K;
  const bool use_c = method == XL_JACPCG;
  const bool textbook = use_c && variant == XL_TEXTBOOK;
  const double2* c2 = reinterpret_cast<const double2*>(s.C + b * (int64_t)n2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ int not_hpd;
  if (threadIdx.x == 0) not_hpd = 0;
  __syncthreads();
  for (int j = warp; j < K; j += nw) {
    const int64_t o = b * per + (int64_t)j * n2;
    const double2* q2 = reinterpret_cast<const double2*>(s.Q + o);
    double2* p2 = reinterpret_cast<double2*>(s.P + o);
    double2* x2 = reinterpret_cast<double2*>(s.X + o);
    double2* r2 = reinterpret_cast<double2*>(s.R + o);
    const double rzj = s.rz[b * K + j];
    const bool act = rzj > 0.0;
    double2 qv[PCG_V64], pv[PCG_V64], cv[PCG_V64];
    double curv = 0.0;
#pragma unroll
    for (int t = 0; t < PCG_V64; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        qv[t] = q2[i];
        pv[t] = p2[i];
        cv[t] = use_c ? c2[i] : make_double2(1.0, 1.0);
        if (use_c && !textbook) { qv[t].x /= cv[t].x; qv[t].y /= cv[t].y; }
        curv += pv[t].x * qv[t].x + pv[t].y * qv[t].y;
      }
    }
    curv = warp_sum_d(curv);
    if (curv <= 0.0 && act && lane == 0) not_hpd = 1;
    const double al = act ? rzj / (curv > 0.0 ? curv : 1.0) : 0.0;
    double acc = 0.0;
    double2 rv[PCG_V64];
#pragma unroll
    for (int t = 0; t < PCG_V64; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        double2 xv = x2[i];
        rv[t] = r2[i];
        xv.x += al * pv[t].x; xv.y += al * pv[t].y;
        rv[t].x -= al * qv[t].x; rv[t].y -= al * qv[t].y;
        x2[i] = xv;
        r2[i] = rv[t];
        acc += textbook ? rv[t].x * (rv[t].x / cv[t].x) + rv[t].y * (rv[t].y / cv[t].y)
                        : rv[t].x * rv[t].x + rv[t].y * rv[t].y;
      }
    }
    acc = warp_sum_d(acc);
    const double be = act ? acc / rzj : 0.0;
#pragma unroll
    for (int t = 0; t < PCG_V64; ++t) {
      const int i = lane + 32 * t;
      if (i < nq) {
        double2 m;
        m.x = (textbook ? rv[t].x / cv[t].x : rv[t].x) + be * pv[t].x;
        m.y = (textbook ? rv[t].y / cv[t].y : rv[t].y) + be * pv[t].y;
        p2[i] = m;
      }
    }
    if (lane == 0) s.rz[b * K + j] = acc;
  }
  __syncthreads();
  if (not_hpd && threadIdx.x == 0 && status[b] == 0) status[b] = XL_STATUS_NOT_HPD;
}

// column-major complex (column j contiguous) -> row-major K x K, 32 x 32 tiles;
// with Q given: GX = Q - xi X and the Re tr(X^H GX) partials per tile
__global__ void __launch_bounds__(256) cm_to_rm64_kernel(const double* __restrict__ Xs, const double* __restrict__ Qs,
                                                         int K, const double* __restrict__ xi_b, double xi,
                                                         double2* __restrict__ out, double* __restrict__ part) {
  const int64_t b = blockIdx.x;
  const int64_t per = 2 * (int64_t)K * K;
  const int i0 = blockIdx.z * XT, j0 = blockIdx.y * XT;
  const double x0 = Qs ? (xi_b ? xi_b[b] : xi) : 0.0;
  __shared__ double2 t[XT][XT + 1];
  double local = 0.0;
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int tj = e / XT, ti = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) {
      const int64_t o = b * per + (int64_t)j * 2 * K + 2 * i;
      const double xr = Xs[o], xim = Xs[o + 1];
      if (Qs) {
        const double gr = Qs[o] - x0 * xr, gi = Qs[o + 1] - x0 * xim;
        t[tj][ti] = make_double2(gr, gi);
        local += xr * gr + xim * gi;
      } else {
        t[tj][ti] = make_double2(xr, xim);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int ti = e / XT, tj = e % XT, i = i0 + ti, j = j0 + tj;
    if (i < K && j < K) out[b * (int64_t)K * K + (int64_t)i * K + j] = t[tj][ti];
  }
  if (part) {
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tt = 0.0;
      for (int w = 0; w < 8; ++w) tt += red[w];
      part[b * gridDim.y * gridDim.z + blockIdx.z * gridDim.y + blockIdx.y] = tt;
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

bool tc_pcg_supported(int K) { return K % 2 == 0 && 2 * K <= 32 * 4 * PCG_V; }

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
    // A = H^H H + xi I on the FP64 tensor cores (dmma.cu): lower-triangle tiles,
    // written with their conjugate mirror -- Hermitian by construction
    return zgemm_dmma(1, H, (int64_t)M * K, K, 0, H, (int64_t)M * K, K, A, (int64_t)K * K, K, K, K, M, Bc, 2,
                      nullptr, nullptr, xi_b, xi, st);
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
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  gram_extract_kernel<<<dim3((unsigned)Bc, nt, nt), 256, 0, st>>>(U, (float2*)A, K, xi_b, xi);
  return check_launch("tc gram extract");
}

// A = (U + U^T)/2 re-assembled as the complex Hermitian H^H H + xi I from the
// fp32 real Gram U of Bc realizations (stream_tc.cu's Gram uses it too)
int tc_gram_extract(const float* U, int64_t Bc, int K, const double* xi_b, double xi, void* A, cudaStream_t st) {
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  gram_extract_kernel<<<dim3((unsigned)Bc, nt, nt), 256, 0, st>>>(U, (float2*)A, K, xi_b, xi);
  return check_launch("tc gram extract");
}
size_t tc_cublas_ws_bytes() { return CUBLAS_WS; }

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
    // W = beta H X (F = H X) on the FP64 tensor cores (dmma.cu)
    return zgemm_dmma(0, H, (int64_t)M * K, K, 0, X, (int64_t)K * K, K, W, (int64_t)M * K, K, M, K, K, Bc, 1, beta,
                      F, nullptr, 0.0, st);
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
  embed_x_kernel<<<dim3((unsigned)Bc, (unsigned)(n2 < 128 ? n2 : 128)), 256, 0, st>>>((const float2*)X, beta, E1, E2, K);
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


size_t tc_pcg_ws_bytes(int64_t B, int K) {
  const size_t n2 = 2 * (size_t)K;
  return align_up((size_t)B * n2 * 2 * n2 * 4) + align_up((size_t)B * n2 * n2 * 4) +
         align_up((size_t)B * 2 * n2 * K * 4) + 4 * align_up((size_t)B * n2 * K * 4) +
         align_up((size_t)B * n2 * 4) + align_up((size_t)B * K * 4);
}

// X ~= A^{-1} for B realizations (complex64, identity RHS, w0 = 0, T iterations);
// status gets NotHpd / Splitting like pcg_kernel.  cws: the CUBLAS_WS bytes
// shared with tc_gram / tc_apply; bufs: tc_pcg_ws_bytes(B, K).
int tc_pcg(int method, int variant, const void* A, int64_t B, int K, int T, void* X, int32_t* status, void* cws,
           void* bufs, cudaStream_t st) {
  cublasHandle_t h = handle_for_device();
  if (!h) { set_error("cublasCreate failed"); return XL_ERR_CUDA; }
  cublasSetStream(h, st);
  cublasSetWorkspace(h, cws, CUBLAS_WS);
  char* p = (char*)bufs;
  const int n2 = 2 * K;
  const PcgState s = pcg_state(p, B, K);
  pcg_init_kernel<<<(unsigned)B, 256, 0, st>>>((const float2*)A, s, K, method, variant, status);
  if (int e = check_launch("tc pcg init")) return e;
  const float one = 1.0f, zero = 0.0f;
  for (int t = 1; t <= T; ++t) {
    // Q = [A''h | A''h] [Ph ; Pl] + A''l Ph
    int e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, K, 2 * n2, &one, s.E1, CUDA_R_32F,
                                                    n2, (long long)n2 * 2 * n2, s.SP, CUDA_R_32F, 2 * n2,
                                                    (long long)2 * n2 * K, &zero, s.Q, CUDA_R_32F, n2,
                                                    (long long)n2 * K, (int)B, CUBLAS_COMPUTE_32F_FAST_TF32,
                                                    CUBLAS_GEMM_DEFAULT),
                         "tc pcg hh+hl");
    if (e) return e;
    e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, K, n2, &one, s.E2, CUDA_R_32F, n2,
                                                (long long)n2 * n2, s.SP, CUDA_R_32F, 2 * n2, (long long)2 * n2 * K,
                                                &one, s.Q, CUDA_R_32F, n2, (long long)n2 * K, (int)B,
                                                CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                     "tc pcg lh");
    if (e) return e;
    pcg_update_kernel<<<(unsigned)B, 256, 0, st>>>(s, K, method, variant, status);
    if ((e = check_launch("tc pcg update"))) return e;
  }
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  pcg_store_x_kernel<<<dim3((unsigned)B, nt, nt), 256, 0, st>>>(s.X, (float2*)X, K);
  return check_launch("tc pcg store");
}


// After tc_pcg (same cws / bufs): GX = (A - xi I) X as complex row-major K x K
// (the coupling up to beta) and the ||F||^2 partials (= Re tr(X^H GX), SURVEY
// K3/K4): ceil(K/32)^2 per realization in part, on the tensor cores.
int tc_gx(const double* xi_b, double xi, int64_t B, int K, void* GX, double* part, void* cws, void* bufs,
          cudaStream_t st) {
  cublasHandle_t h = handle_for_device();
  if (!h) { set_error("cublasCreate failed"); return XL_ERR_CUDA; }
  cublasSetStream(h, st);
  cublasSetWorkspace(h, cws, CUBLAS_WS);
  const int n2 = 2 * K;
  const PcgState s = pcg_state((char*)bufs, B, K);
  const unsigned gx = grid_for((int64_t)n2 * K, 256);
  split_x_kernel<<<dim3((unsigned)B, gx > 64 ? 64 : gx), 256, 0, st>>>(s, K);
  if (int e = check_launch("tc gx split")) return e;
  const float one = 1.0f, zero = 0.0f;
  int e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, K, 2 * n2, &one, s.E1, CUDA_R_32F,
                                                  n2, (long long)n2 * 2 * n2, s.SP, CUDA_R_32F, 2 * n2,
                                                  (long long)2 * n2 * K, &zero, s.Q, CUDA_R_32F, n2,
                                                  (long long)n2 * K, (int)B, CUBLAS_COMPUTE_32F_FAST_TF32,
                                                  CUBLAS_GEMM_DEFAULT),
                       "tc gx hh+hl");
  if (e) return e;
  e = cublas_check(cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, K, n2, &one, s.E2, CUDA_R_32F, n2,
                                              (long long)n2 * n2, s.SP, CUDA_R_32F, 2 * n2, (long long)2 * n2 * K,
                                              &one, s.Q, CUDA_R_32F, n2, (long long)n2 * K, (int)B,
                                              CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                   "tc gx lh");
  if (e) return e;
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  gx_finish_kernel<<<dim3((unsigned)B, nt, nt), 256, 0, st>>>(s, K, xi_b, xi, (float2*)GX, part);
  return check_launch("tc gx finish");
}


size_t tc_pcg64_ws_bytes(int64_t B, int K) {
  const size_t n2 = 2 * (size_t)K;
  return 4 * align_up((size_t)B * n2 * K * 8) + align_up((size_t)B * n2 * 8) + align_up((size_t)B * K * 8);
}

bool tc_pcg64_supported(int K) { return 2 * K <= 32 * 2 * PCG_V64; }

// complex128 Jac-PCG / CG for the rzf path (identity RHS, w0 = 0, T iterations):
// Q = A P per iteration as one ZGEMM (OP_T of the column-major view of row-major
// A is A), then the per-column update; X out row-major.
int tc_pcg64(int method, int variant, const void* A, int64_t B, int K, int T, void* X, int32_t* status, void* cws,
             void* bufs, cudaStream_t st) {
  (void)cws;
  const PcgState64 s = pcg_state64((char*)bufs, B, K);
  pcg_init64_kernel<<<(unsigned)B, 256, 0, st>>>((const double2*)A, s, K, method, variant, status);
  if (int e = check_launch("tc pcg64 init")) return e;
  const long long sk = (long long)K * K;
  for (int t = 1; t <= T; ++t) {
    // column-major Q = A P: in row-major views Q^T = P^T A^T (dmma.cu, opB = T)
    int e = zgemm_dmma(0, s.P, sk, K, 1, A, sk, K, s.Q, sk, K, K, K, K, B, 0, nullptr, nullptr, nullptr, 0.0, st);
    if (e) return e;
    pcg_update64_kernel<<<(unsigned)B, 256, 0, st>>>(s, K, method, variant, status);
    if ((e = check_launch("tc pcg64 update"))) return e;
  }
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  cm_to_rm64_kernel<<<dim3((unsigned)B, nt, nt), 256, 0, st>>>(s.X, nullptr, K, nullptr, 0.0, (double2*)X, nullptr);
  return check_launch("tc pcg64 store");
}

// After tc_pcg64: GX = (A - xi I) X and the ||F||^2 partials per 32 x 32 tile.
int tc_gx64(const void* A, const double* xi_b, double xi, int64_t B, int K, void* GX, double* part, void* cws,
            void* bufs, cudaStream_t st) {
  (void)cws;
  const PcgState64 s = pcg_state64((char*)bufs, B, K);
  const long long sk = (long long)K * K;
  int e = zgemm_dmma(0, s.X, sk, K, 1, A, sk, K, s.Q, sk, K, K, K, K, B, 0, nullptr, nullptr, nullptr, 0.0, st);
  if (e) return e;
  const unsigned nt = (unsigned)((K + XT - 1) / XT);
  cm_to_rm64_kernel<<<dim3((unsigned)B, nt, nt), 256, 0, st>>>(s.X, s.Q, K, xi_b, xi, (double2*)GX, part);
  return check_launch("tc gx64 finish");
}

}  // namespace xl
