// Aspect ratios of a tagging plan on the GPU (ref/tagging.py:110-123 via
// :355-379): rho_i = max_j |t_j . z_i| / min_j |t_j . z_i| over the far field
// j of block i (j not a neighbour of i), 1 if the max is 0, inf if the min is
// 0, NaN when the far field is empty. The reference forms the b x b matrix
// |T Z^T| on the host; for b = 4096 (config 5) that product and its
// reductions took ~70-370 ms per draw of the redraw policy, on the GPU it is
// one launch per draw. One CTA per block i; the near set is a shared-memory
// bitmask; the dot products run in column order with fma.
#include <cmath>

#include "common.cuh"
#include "nullvec.cuh"

namespace ublr {
namespace {

constexpr int TA_THREADS = 256;

__global__ void __launch_bounds__(TA_THREADS) k_tag_aspect(const double* __restrict__ T, const double* __restrict__ Z,
                                                           int ell, const int32_t* __restrict__ nptr,
                                                           const int32_t* __restrict__ nidx, int b,
                                                           double* __restrict__ rho) {
  extern __shared__ uint32_t near_bits[];
  __shared__ double red_lo[TA_THREADS / 32], red_hi[TA_THREADS / 32];
  __shared__ double zi[32];
  const int i = blockIdx.x;
  const int words = (b + 31) / 32;
  for (int w = threadIdx.x; w < words; w += TA_THREADS) near_bits[w] = 0u;
  if (threadIdx.x < ell) zi[threadIdx.x] = Z[(int64_t)i * ell + threadIdx.x];
  __syncthreads();
  const int p0 = nptr[i], p1 = nptr[i + 1];
  for (int p = p0 + threadIdx.x; p < p1; p += TA_THREADS) atomicOr(&near_bits[nidx[p] >> 5], 1u << (nidx[p] & 31));
  __syncthreads();
  double lo = INFINITY, hi = -INFINITY;
  for (int j = threadIdx.x; j < b; j += TA_THREADS) {
    if (near_bits[j >> 5] & (1u << (j & 31))) continue;
    const double* tj = T + (int64_t)j * ell;
    double s = 0.0;
    for (int c = 0; c < ell; ++c) s = fma(tj[c], zi[c], s);
    s = fabs(s);
    lo = fmin(lo, s);
    hi = fmax(hi, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red_lo[warp] = lo;
    red_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < TA_THREADS / 32; ++w) {
      lo = fmin(lo, red_lo[w]);
      hi = fmax(hi, red_hi[w]);
    }
    double r;
    if (p1 - p0 >= b) r = NAN;              // empty far field
    else if (hi == 0.0) r = 1.0;
    else if (lo == 0.0) r = INFINITY;
    else r = hi / lo;
    rho[i] = r;
  }
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_tag_aspect(const double* T, const double* Z, int ell, const int32_t* nptr, const int32_t* nidx,
                               int b, double* rho, void* stream) {
  UBLR_REQUIRE(T && Z && nptr && nidx && rho && b > 0 && ell >= 1 && ell <= 32, UBLR_ERR_VALUE,
               "ublr_tag_aspect: bad arguments (ell <= 32)");
  size_t sm = (size_t)((b + 31) / 32) * sizeof(uint32_t);
  UBLR_REQUIRE(sm <= 48 * 1024, UBLR_ERR_VALUE, "ublr_tag_aspect: b too large for the near-set bitmask");
  k_tag_aspect<<<b, TA_THREADS, sm, (cudaStream_t)stream>>>(T, Z, ell, nptr, nidx, b, rho);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

// Device twin of ublr_null_vectors (same arithmetic, same bits: nullvec.cuh),
// one thread per row set. Lets the pipeline launch the block QR right after
// the sketch while the host evaluates the same plan for its redraw decision.
namespace ublr {
namespace {
__global__ void k_null_vectors(const double* __restrict__ T, int ell, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ idx, int nsets, double* __restrict__ Z,
                               double* __restrict__ res) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsets) return;
  double A[ublr::nullvec::MAX_ELL * ublr::nullvec::MAX_ELL], tau[ublr::nullvec::MAX_ELL];
  const int r0 = ptr[s], sz = ptr[s + 1] - r0;
  if (sz >= ell) {   // no null vector (the host planner raises DegenerateTagsError)
    for (int i = 0; i < ell; ++i) Z[(int64_t)s * ell + i] = 0.0;
    res[s] = INFINITY;
    return;
  }
  res[s] = ublr::nullvec::null_vector(T, ell, idx + r0, sz, A, tau, Z + (int64_t)s * ell);
}
}  // namespace
}  // namespace ublr

extern "C" int ublr_null_vectors_device(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int nsets,
                                        double* Z, double* res, void* stream) {
  UBLR_REQUIRE(T && ell >= 1 && ell <= ublr::nullvec::MAX_ELL && ptr && idx && nsets >= 0 && Z && res,
               UBLR_ERR_VALUE, "ublr_null_vectors_device: bad arguments (ell <= 32)");
  if (nsets == 0) return UBLR_OK;
  ublr::k_null_vectors<<<(nsets + 63) / 64, 64, 0, (cudaStream_t)stream>>>(T, ell, ptr, idx, nsets, Z, res);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
