// Batched complex128 GEMM on the FP64 tensor cores (DMMA, mma.sync m8n8k4
// f64) for the large-K general path: the products of gram_regularized
// (precoder.py:59-60: A = H^H H, Hermitian by construction, + xi I),
// rzf_iterative's F = H X (precoder.py:90, beta folded in) and the Jac-PCG /
// CG products Q = A P (linsolve.py:275) -- replacing library ZGEMM.
//
// C[b] = op(A[b]) op(B[b]), row-major complex128:
//   opA = N: A stored [m][k] (lda); opA = C: A stored [k][m], used conjugated
//   (A^H); opB = N: B stored [k][n]; opB = T: B stored [n][k] (transposed).
// CTA tile 64 x 64, K chunk 16, 8 warps as 2 (m) x 4 (n) of 32 x 16; the tiles
// are staged through registers into shared memory as [k][m] / [k][n] planes
// (prefetch of chunk c + 1 overlaps the DMMAs of chunk c).  Each 8 x 8 x 4
// complex block is four real DMMAs (Re += Ar Br - Ai Bi, Im += Ar Bi + Ai Br)
// with fp64 accumulation; complex multiply-adds in a fixed order, so results
// are deterministic.
//
// Epilogues: STORE (C = acc), SCALE (C = beta[b] acc, F = acc optional), and
// HERM for the Gram: only tiles on or below the diagonal are computed; entry
// (i, j), i > j, is written with its conjugate mirror (j, i), the diagonal as
// Re + xi (imaginary part 0) -- Hermitian by construction.
#include <stdint.h>

#include "xl_common.cuh"

namespace xl {
namespace dm {

constexpr int TM = 64, TN = 64, TK = 16, NT = 256;
enum { OP_N = 0, OP_C = 1, OP_T = 1 };
enum { EPI_STORE = 0, EPI_SCALE = 1, EPI_HERM = 2 };

struct Args {
  const double2* A; int64_t sA; int lda; int opA;
  const double2* B; int64_t sB; int ldb; int opB;
  double2* C; int64_t sC; int ldc;
  double2* F;                 // EPI_SCALE: optional unscaled copy
  int M, N, K;
  int epi;
  const double* beta;         // EPI_SCALE: per batch
  const double* xi_b; double xi;  // EPI_HERM
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// element (r, k) of the A tile / (k, c) of the B tile, zero outside the matrix
__device__ __forceinline__ double2 ldA(const Args& g, const double2* A, int r, int k) {
  if (r >= g.M || k >= g.K) return make_double2(0.0, 0.0);
  return g.opA == OP_N ? A[(int64_t)r * g.lda + k] : A[(int64_t)k * g.lda + r];
}
__device__ __forceinline__ double2 ldB(const Args& g, const double2* B, int k, int c) {
  if (k >= g.K || c >= g.N) return make_double2(0.0, 0.0);
  return g.opB == OP_N ? B[(int64_t)k * g.ldb + c] : B[(int64_t)c * g.ldb + k];
}

constexpr int SMEM = 2 * 2 * TK * (TM + 1) * (int)sizeof(double2);  // 66.5 KiB (TM == TN)

__global__ void __launch_bounds__(NT, 2) zgemm_kernel(Args g) {
  // [buf][k][m + 1]: the +1 spreads the transposing stores and the fragment loads over the banks
  extern __shared__ __align__(16) double2 dsm[];
  double2 (*sA)[TK][TM + 1] = reinterpret_cast<double2 (*)[TK][TM + 1]>(dsm);
  double2 (*sB)[TK][TN + 1] = reinterpret_cast<double2 (*)[TK][TN + 1]>(dsm + 2 * TK * (TM + 1));
  const int64_t b = blockIdx.z;
  int tm = blockIdx.y, tn = blockIdx.x;
  if (g.epi == EPI_HERM) {  // lower-triangle tiles: blockIdx.x enumerates (tm >= tn)
    const int t = blockIdx.x;
    tm = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((tm + 1) * (tm + 2) / 2 <= t) ++tm;
    while (tm * (tm + 1) / 2 > t) --tm;
    tn = t - tm * (tm + 1) / 2;
  }
  const int m0 = tm * TM, n0 = tn * TN;
  const double2* A = g.A + b * g.sA;
  const double2* Bm = g.B + b * g.sB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile rows 32 wm.., cols 16 wn..
  const bool conjA = g.opA == OP_C;

  // global -> register staging: 4 elements of A and 4 of B per thread per chunk
  // A tile element e = tid + 256 i (i < 4): opA N: (r = e / 16, k = e % 16) (rows of
  // 16 contiguous complex); opA C: (k = e / 64, r = e % 64) (rows of 64)
  double2 ra[4], rb[4];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + NT * i;
      if (g.opA == OP_N) ra[i] = ldA(g, A, m0 + e / TK, k0 + e % TK);
      else ra[i] = ldA(g, A, m0 + e % TM, k0 + e / TM);
      if (g.opB == OP_N) rb[i] = ldB(g, Bm, k0 + e / TN, n0 + e % TN);
      else rb[i] = ldB(g, Bm, k0 + e % TK, n0 + e / TK);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + NT * i;
      if (g.opA == OP_N) sA[buf][e % TK][e / TK] = ra[i];
      else sA[buf][e / TM][e % TM] = ra[i];
      if (g.opB == OP_N) sB[buf][e / TN][e % TN] = rb[i];
      else sB[buf][e % TK][e / TK] = rb[i];
    }
  };

  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) cr[x][y][0] = cr[x][y][1] = ci[x][y][0] = ci[x][y][1] = 0.0;

  const int nk = (g.K + TK - 1) / TK;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int c = 0; c < nk; ++c) {
    const int buf = c & 1;
    if (c + 1 < nk) fetch((c + 1) * TK);
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      const int k = kk + (lane & 3);
      double ar[4], ai[4], br[2], bi[2];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const double2 v = sA[buf][k][32 * wm + 8 * x + (lane >> 2)];
        ar[x] = v.x;
        ai[x] = conjA ? -v.y : v.y;
      }
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const double2 v = sB[buf][k][16 * wn + 8 * y + (lane >> 2)];
        br[y] = v.x;
        bi[y] = v.y;
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          dmma(cr[x][y], ar[x], br[y]);
          dmma(cr[x][y], -ai[x], bi[y]);
          dmma(ci[x][y], ar[x], bi[y]);
          dmma(ci[x][y], ai[x], br[y]);
        }
    }
    if (c + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }

  // ---- epilogue: thread holds C[row][col], C[row][col + 1] of each 8 x 8 block
  double2* C = g.C + b * g.sC;
  const double bt = g.epi == EPI_SCALE ? g.beta[b] : 1.0;
  const double xi = g.epi == EPI_HERM ? (g.xi_b ? g.xi_b[b] : g.xi) : 0.0;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      const int row = m0 + 32 * wm + 8 * x + (lane >> 2);
      const int col = n0 + 16 * wn + 8 * y + 2 * (lane & 3);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = col + e;
        if (row >= g.M || cc >= g.N) continue;
        const double re = cr[x][y][e], im = ci[x][y][e];
        if (g.epi == EPI_HERM) {
          if (row == cc) {
            C[(int64_t)row * g.ldc + cc] = make_double2(re + xi, 0.0);
          } else if (row > cc) {
            C[(int64_t)row * g.ldc + cc] = make_double2(re, im);
            C[(int64_t)cc * g.ldc + row] = make_double2(re, -im);
          }
        } else {
          C[(int64_t)row * g.ldc + cc] = make_double2(bt * re, bt * im);
          if (g.F) g.F[b * g.sC + (int64_t)row * g.ldc + cc] = make_double2(re, im);
        }
      }
    }
}

}  // namespace dm

// row-major complex128 C[b] = op(A[b]) op(B[b]) (see dm::Args)
int zgemm_dmma(int opA, const void* A, int64_t sA, int lda, int opB, const void* B, int64_t sB, int ldb, void* C,
               int64_t sC, int ldc, int M, int N, int K, int64_t batch, int epi, const double* beta, void* F,
               const double* xi_b, double xi, cudaStream_t st) {
  if (batch <= 0) return XL_SUCCESS;
  if (batch > 65535) {  // grid.z limit: split
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
      if (int e = zgemm_dmma(opA, (const double2*)A + b0 * sA, sA, lda, opB, (const double2*)B + b0 * sB, sB, ldb,
                             (double2*)C + b0 * sC, sC, ldc, M, N, K, nb, epi, beta ? beta + b0 : nullptr,
                             F ? (double2*)F + b0 * sC : nullptr, xi_b ? xi_b + b0 : nullptr, xi, st))
        return e;
    }
    return XL_SUCCESS;
  }
  dm::Args g{(const double2*)A, sA, lda, opA, (const double2*)B, sB, ldb, opB, (double2*)C, sC, ldc, (double2*)F,
             M, N, K, epi, beta, xi_b, xi};
  const int gm = (M + dm::TM - 1) / dm::TM, gn = (N + dm::TN - 1) / dm::TN;
  dim3 grid = epi == dm::EPI_HERM ? dim3((unsigned)(gm * (gm + 1) / 2), 1, (unsigned)batch)
                                  : dim3((unsigned)gn, (unsigned)gm, (unsigned)batch);
  cudaFuncSetAttribute(dm::zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dm::SMEM);
  dm::zgemm_kernel<<<grid, dm::NT, dm::SMEM, st>>>(g);
  return check_launch("zgemm dmma");
}

}  // namespace xl
