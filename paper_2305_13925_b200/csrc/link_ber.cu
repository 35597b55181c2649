// BER detection chain of ber_montecarlo (metrics.py:124-140), batched over
// channel draws: Y = Bc s + n with s = QPSK(bits) (metrics.py:73-77), genie
// scaling by the diagonal gain (zero gain -> 1, metrics.py:134-135), hard
// decisions (metrics.py:80-83) and the bit-error count per draw.
//
// One thread per (user k, symbol n); a warp spans 32 consecutive symbols of
// one user, so the coupling row Bc[k, :] is a warp-uniform (broadcast) load
// and the bit pairs / noise are coalesced.  Error counts are integer atomics:
// order-independent, so the result is deterministic.
#include "xl_common.cuh"

namespace xl {

namespace {

constexpr int BX = 32, BY = 8;  // symbols x users per CTA

// numpy's complex division (Smith's scaling, multiply by the reciprocal)
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

template <typename R>
__global__ void __launch_bounds__(BX * BY)
ber_kernel(const cplx<R>* __restrict__ Bc, const int8_t* __restrict__ bits,
           const cplx<R>* __restrict__ noise, int K, int nsym, unsigned long long* errors) {
  using C = cplx<R>;
  const int64_t b = blockIdx.z;
  const int n = blockIdx.x * BX + threadIdx.x, k = blockIdx.y * BY + threadIdx.y;
  int err = 0;
  if (n < nsym && k < K) {
    const C* row = Bc + (b * K + k) * (int64_t)K;
    const char2* bp = reinterpret_cast<const char2*>(bits) + b * (int64_t)K * nsym;
    // (1 - 2 b) / sqrt(2) exactly as numpy: a real divisor becomes a multiply
    // by the rounded reciprocal (complex division with rat = 0)
    const R scl = (R)1 / sqrt((R)2);
    C y = noise[(b * K + k) * (int64_t)nsym + n];
    C acc = mk<R>(0, 0);
    for (int j = 0; j < K; ++j) {
      const char2 bj = bp[(int64_t)j * nsym + n];
      const C s = mk<R>(((R)1 - (R)2 * (R)bj.x) * scl, ((R)1 - (R)2 * (R)bj.y) * scl);
      cfma(acc, row[j], s);
    }
    y = cadd(acc, y);
    C g = row[k];
    if (g.x == (R)0 && g.y == (R)0) g = mk<R>(1, 0);  // dead user: coin flips
    const C z = cdiv_np<R>(y, g);
    const char2 own = bp[(int64_t)k * nsym + n];
    err = (int)((z.x < (R)0) != (own.x != 0)) + (int)((z.y < (R)0) != (own.y != 0));
  }
  // CTA sum, one atomic per CTA
  for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
  __shared__ int part[BY];
  if (threadIdx.x == 0) part[threadIdx.y] = err;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    int t = 0;
    for (int i = 0; i < BY; ++i) t += part[i];
    if (t) atomicAdd(errors + b, (unsigned long long)t);
  }
}

}  // namespace

int launch_ber(int dtype, const void* Bc, const int8_t* bits, const void* noise, int64_t B, int K,
               int nsym, int64_t* errors, cudaStream_t st) {
  if (cudaMemsetAsync(errors, 0, (size_t)B * sizeof(int64_t), st) != cudaSuccess) return check_launch("ber memset");
  const dim3 blk(BX, BY);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    const dim3 grid((unsigned)((nsym + BX - 1) / BX), (unsigned)((K + BY - 1) / BY), (unsigned)nb);
    unsigned long long* e = reinterpret_cast<unsigned long long*>(errors + b0);
    const int8_t* bb = bits + b0 * (int64_t)K * nsym * 2;
    if (dtype == XL_C64)
      ber_kernel<float><<<grid, blk, 0, st>>>((const float2*)Bc + b0 * (int64_t)K * K, bb,
                                              (const float2*)noise + b0 * (int64_t)K * nsym, K, nsym, e);
    else
      ber_kernel<double><<<grid, blk, 0, st>>>((const double2*)Bc + b0 * (int64_t)K * K, bb,
                                               (const double2*)noise + b0 * (int64_t)K * nsym, K, nsym, e);
    if (int rc = check_launch("ber")) return rc;
  }
  return XL_SUCCESS;
}

}  // namespace xl
