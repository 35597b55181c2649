// Fused complex128 precoder for small K (K in {16, 32}, H of one realization
// resident in shared memory): one CTA per realization runs the whole chain of
// rzf_iterative + sinr_eq9 on chip with every product on the FP64 tensor
// cores (DMMA, mma.sync m8n8k4 f64):
//
//   A = H^H H + xi I          gram_regularized (precoder.py:53-61): antennas
//                             split over the 8 warps, partial tiles summed in
//                             warp order (deterministic), lower triangle +
//                             conjugate mirror (Hermitian by construction)
//   Jac-PCG / CG, T iters     _pcg_textbook / _pcg_core (linsolve.py:217-294)
//                             on the K identity right-hand sides: Q = A P on
//                             DMMA, per-column scalars in fixed order
//   GX = (A - xi I) X         ||F||^2 = Re tr(X^H GX) (precoder.py:64-70 with
//                             F = H X, the K x K form), beta = sqrt(P / ||F||^2)
//   W = beta H X              (precoder.py:90) on DMMA, F = H X optional
//   B = beta GX = H^H W       coupling_matrix + sinr_eq9 (metrics.py:35-58)
//
// This replaces the general path's seven SIMT launches for cfg1 (configs[0]:
// M = 256, K = 16, complex128) with one.
#include <math.h>
#include <stdint.h>

#include "xl_common.cuh"

namespace xl {
namespace fc {

constexpr int NT = 256, NW = NT / 32;
constexpr int MAX_SMEM = 200 * 1024;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// complex 8x8x4 block: (cr, ci) += (ar + i ai) (br + i bi)
__device__ __forceinline__ void cmma(double (&cr)[2], double (&ci)[2], double ar, double ai, double br, double bi) {
  dmma(cr, ar, br);
  dmma(cr, -ai, bi);
  dmma(ci, ar, bi);
  dmma(ci, ai, br);
}

struct Params {
  const double2* H;
  int64_t B;
  int M, method, variant, T;
  double xi;
  const double* xi_b;
  double power, sigma2;
  double2 *W, *F, *X;
  double *beta, *gamma, *sum_se;
  int32_t* status;
};

// C (K x K, smem, row-major) = Aop * Bm where Aop = A or A - s I ... computed by
// warps over 8 x 8 output tiles; a, b row-major K x K in smem.
template <int K>
__device__ __forceinline__ void kxk_product(const double2* a, const double2* b, double2* c, double diag_shift) {
  constexpr int NTL = K / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tile = warp; tile < NTL * NTL; tile += NW) {
    const int ti = tile / NTL, tj = tile % NTL;
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
#pragma unroll
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int r = 8 * ti + (lane >> 2), kk = k0 + (lane & 3), cc = 8 * tj + (lane >> 2);
      double2 av = a[r * K + kk];
      if (r == kk) av.x -= diag_shift;
      const double2 bv = b[kk * K + cc];
      cmma(cr, ci, av.x, av.y, bv.x, bv.y);
    }
    const int r = 8 * ti + (lane >> 2), cc = 8 * tj + 2 * (lane & 3);
    c[r * K + cc] = make_double2(cr[0], ci[0]);
    c[r * K + cc + 1] = make_double2(cr[1], ci[1]);
  }
}

template <int K>
__global__ void __launch_bounds__(NT) fused_c128_kernel(Params p) {
  extern __shared__ __align__(16) double2 smem[];
  const int M = p.M;
  double2* Hs = smem;                    // [M][K]
  double2* As = Hs + (size_t)M * K;      // [K][K]
  double2* Xs = As + K * K;              // solver state, [K][K] each (row i, column j)
  double2* Rs = Xs + K * K;
  double2* Ps = Rs + K * K;
  double2* Qs = Ps + K * K;
  double* cdg = reinterpret_cast<double*>(Qs + K * K);  // [K] Re diag(A) (preconditioner)
  double* rzs = cdg + K;                                  // [K] rz per column
  double* coef = rzs + K;                                 // [K] alpha / beta per column
  double* icd = coef + K;                                 // [K] 1 / cdg (computed once)
  double* red = icd + K;                                  // [NW] reductions
  int* flags = reinterpret_cast<int*>(red + NW);          // [0] not_hpd
  constexpr int NTL = K / 8;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool use_c = p.method == XL_JACPCG;
  const bool textbook = use_c && p.variant == XL_TEXTBOOK;
  const double xi = p.xi_b ? p.xi_b[b] : p.xi;

  // ---- H -> smem (16-B cp.async: every load in flight at once, not one DRAM
  // round trip per loop trip)
  const double2* Hb = p.H + b * (int64_t)M * K;
  for (int e = tid; e < M * K; e += NT)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(Hs + e)),
                 "l"(Hb + e)
                 : "memory");
  if (tid == 0) flags[0] = 0;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // ---- Gram: warp w sums antennas [w M/8, (w+1) M/8) for every 8 x 8 tile
  {
    double gr[NTL * NTL][2], gi[NTL * NTL][2];
#pragma unroll
    for (int t = 0; t < NTL * NTL; ++t) gr[t][0] = gr[t][1] = gi[t][0] = gi[t][1] = 0.0;
    const int a0 = warp * (M / NW), a1 = a0 + M / NW;
    for (int a = a0; a < a1; a += 4) {
      const int aa = a + (lane & 3);
      double hr[NTL], hi[NTL];  // fragment values H[aa][8 t + lane/4]
#pragma unroll
      for (int t = 0; t < NTL; ++t) {
        const double2 v = Hs[aa * K + 8 * t + (lane >> 2)];
        hr[t] = v.x;
        hi[t] = v.y;
      }
#pragma unroll
      for (int ti = 0; ti < NTL; ++ti)
#pragma unroll
        for (int tj = 0; tj < NTL; ++tj)  // (H^H)[i][a] = conj(H[a][i])
          cmma(gr[ti * NTL + tj], gi[ti * NTL + tj], hr[ti], -hi[ti], hr[tj], hi[tj]);
    }
    // fixed warp order: warp 0 stores, warps 1..7 add in turn
    for (int w = 0; w < NW; ++w) {
      if (warp == w) {
#pragma unroll
        for (int t = 0; t < NTL * NTL; ++t) {
          const int r = 8 * (t / NTL) + (lane >> 2), c = 8 * (t % NTL) + 2 * (lane & 3);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double2 v = w == 0 ? make_double2(0.0, 0.0) : As[r * K + c + e];
            v.x += gr[t][e];
            v.y += gi[t][e];
            As[r * K + c + e] = v;
          }
        }
      }
      __syncthreads();
    }
  }
  // Hermitian by construction: the lower triangle and its mirror; real diagonal + xi
  for (int e = tid; e < K * K; e += NT) {
    const int i = e / K, j = e % K;
    if (i < j) As[e] = make_double2(As[j * K + i].x, -As[j * K + i].y);
  }
  __syncthreads();
  if (tid < K) {
    As[tid * K + tid] = make_double2(As[tid * K + tid].x + xi, 0.0);
    cdg[tid] = As[tid * K + tid].x;
    icd[tid] = 1.0 / cdg[tid];
  }
  __syncthreads();
  // zero preconditioner diagonal -> Splitting (linsolve.py:205-208)
  if (tid == 0 && use_c) {
    for (int i = 0; i < K; ++i)
      if (cdg[i] == 0.0) flags[0] |= 2;
  }

  // ---- initial state (linsolve.py:224-229, 264-268): w = 0, r = I (Algorithm 1:
  // C^-1 I), m = z
  for (int e = tid; e < K * K; e += NT) {
    const int i = e / K, j = e % K;
    const double ei = (i == j) ? 1.0 : 0.0;
    const double ic = use_c ? icd[i] : 1.0;
    const double r = (use_c && !textbook) ? ei * ic : ei;
    Xs[e] = make_double2(0.0, 0.0);
    Rs[e] = make_double2(r, 0.0);
    Ps[e] = make_double2(textbook ? ei * ic : r, 0.0);
  }
  __syncthreads();
  // rz_j = Re(r_j^H z_j): identity columns, z = r / c (textbook), r (CG / Algorithm 1)
  if (tid < K) {
    const double ic = use_c ? icd[tid] : 1.0;
    rzs[tid] = textbook ? ic : (use_c ? ic * ic : 1.0);
  }
  __syncthreads();

  for (int t = 1; t <= p.T; ++t) {
    // Q = A m (Algorithm 1: z = C^-1 A m)
    kxk_product<K>(As, Ps, Qs, 0.0);
    __syncthreads();
    if (use_c && !textbook)
      for (int e = tid; e < K * K; e += NT) {
        const double ic = icd[e / K];
        Qs[e] = make_double2(Qs[e].x * ic, Qs[e].y * ic);
      }
    __syncthreads();
    // curvature per column (linsolve.py:276, 240): Re(m^H z), rows in order
    if (tid < K) {
      const int j = tid;
      double curv = 0.0;
      for (int i = 0; i < K; ++i) {
        const double2 m = Ps[i * K + j], z = Qs[i * K + j];
        curv += m.x * z.x + m.y * z.y;
      }
      const double rzj = rzs[j];
      const bool act = rzj > 0.0;
      if (curv <= 0.0 && act) atomicOr(flags, 1);
      coef[j] = act ? rzj / (curv > 0.0 ? curv : 1.0) : 0.0;
    }
    __syncthreads();
    // w += alpha m, r -= alpha z
    for (int e = tid; e < K * K; e += NT) {
      const double al = coef[e % K];
      const double2 m = Ps[e], z = Qs[e];
      double2 x = Xs[e], r = Rs[e];
      x.x += al * m.x; x.y += al * m.y;
      r.x -= al * z.x; r.y -= al * z.y;
      Xs[e] = x;
      Rs[e] = r;
    }
    __syncthreads();
    // rz' and beta (linsolve.py:284-288), m = z' + beta m
    if (tid < K) {
      const int j = tid;
      double rn = 0.0;
      for (int i = 0; i < K; ++i) {
        const double2 r = Rs[i * K + j];
        const double ic = textbook ? icd[i] : 1.0;
        rn += r.x * (r.x * ic) + r.y * (r.y * ic);
      }
      const double rzj = rzs[j];
      coef[j] = rzj > 0.0 ? rn / rzj : 0.0;
      rzs[j] = rn;
    }
    __syncthreads();
    for (int e = tid; e < K * K; e += NT) {
      const double be = coef[e % K];
      const double ic = textbook ? icd[e / K] : 1.0;
      const double2 r = Rs[e], m = Ps[e];
      Ps[e] = make_double2(r.x * ic + be * m.x, r.y * ic + be * m.y);
    }
    __syncthreads();
  }

  // ---- GX = (A - xi I) X (in Qs), ||F||^2 = Re tr(X^H GX), beta
  kxk_product<K>(As, Xs, Qs, xi);
  __syncthreads();
  {
    double f = 0.0;
    for (int e = tid; e < K * K; e += NT) {
      const double2 x = Xs[e], g = Qs[e];
      f += x.x * g.x + x.y * g.y;
    }
    f = warp_sum(f);
    if (lane == 0) red[warp] = f;
  }
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < NW; ++w) fro += red[w];
  const bool degenerate = !(fro > 0.0);
  const double bt = degenerate ? 0.0 : sqrt(p.power / fro);

  // ---- W = beta H X (F = H X): 8 x 8 output tiles over the warps
  double2* Wb = p.W + b * (int64_t)M * K;
  double2* Fb = p.F ? p.F + b * (int64_t)M * K : nullptr;
  for (int tile = warp; tile < (M / 8) * NTL; tile += NW) {
    const int tm = tile / NTL, tn = tile % NTL;
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
#pragma unroll
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double2 hv = Hs[(8 * tm + (lane >> 2)) * K + k0 + (lane & 3)];
      const double2 xv = Xs[(k0 + (lane & 3)) * K + 8 * tn + (lane >> 2)];
      cmma(cr, ci, hv.x, hv.y, xv.x, xv.y);
    }
    const int r = 8 * tm + (lane >> 2), c = 8 * tn + 2 * (lane & 3);
    reinterpret_cast<double4*>(Wb + r * K + c)[0] = make_double4(bt * cr[0], bt * ci[0], bt * cr[1], bt * ci[1]);
    if (Fb) reinterpret_cast<double4*>(Fb + r * K + c)[0] = make_double4(cr[0], ci[0], cr[1], ci[1]);
  }
  if (p.X) {
    double2* Xo = p.X + b * (int64_t)K * K;
    for (int e = tid; e < K * K; e += NT) Xo[e] = Xs[e];
  }

  // ---- SINR / SE from B = beta GX (row k: user k; metrics.py:47-58)
  if (warp == 0) {
    double s = 0.0;
    for (int k = lane; k < K; k += 32) {
      double sig = 0.0, intf = 0.0;
      for (int j = 0; j < K; ++j) {
        const double2 g = Qs[k * K + j];
        const double v = bt * bt * (g.x * g.x + g.y * g.y);
        if (j == k) sig = v;
        else intf += v;
      }
      const double gam = sig / (intf + p.sigma2);
      if (p.gamma) p.gamma[b * K + k] = gam;
      s += log2(1.0 + gam);
    }
    s = warp_sum(s);  // fixed butterfly order
    if (lane == 0) {
      p.sum_se[b] = s;
      p.beta[b] = bt;
      int st = 0;
      if (flags[0] & 2) st = XL_STATUS_SPLITTING;
      else if (flags[0] & 1) st = XL_STATUS_NOT_HPD;
      else if (degenerate) st = XL_STATUS_DEGENERATE;
      p.status[b] = st;
    }
  }
}

template <int K>
size_t smem_bytes(int M) {
  return ((size_t)M * K + 5 * K * K) * sizeof(double2) + (4 * K + NW) * sizeof(double) + 16;
}

}  // namespace fc

bool fc128_supported(int dtype, int method, int M, int K) {
  if (dtype != XL_C128 || method == XL_DIRECT || M < 32 || M % 32 != 0) return false;  // 8 warps x k-steps of 4
  if (K == 16) return fc::smem_bytes<16>(M) <= (size_t)fc::MAX_SMEM;
  if (K == 32) return fc::smem_bytes<32>(M) <= (size_t)fc::MAX_SMEM;
  return false;
}

int fc128_rzf(int method, int variant, const void* H, int64_t B, int M, int K, double xi, const double* xi_b,
              double power, int T, double sigma2, void* W, void* F, double* beta, double* gamma, double* sum_se,
              void* X, int32_t* status, cudaStream_t st) {
  fc::Params p{(const double2*)H, B, M, method, variant, T, xi, xi_b, power, sigma2, (double2*)W, (double2*)F,
               (double2*)X, beta, gamma, sum_se, status};
  if (K == 16) {
    const size_t sm = fc::smem_bytes<16>(M);
    cudaFuncSetAttribute(fc::fused_c128_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fc::fused_c128_kernel<16><<<(unsigned)B, fc::NT, sm, st>>>(p);
  } else {
    const size_t sm = fc::smem_bytes<32>(M);
    cudaFuncSetAttribute(fc::fused_c128_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fc::fused_c128_kernel<32><<<(unsigned)B, fc::NT, sm, st>>>(p);
  }
  return check_launch("fused c128");
}

}  // namespace xl
