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
// One warp per row set, the set's ell x sz matrix in shared memory. Every
// sum keeps the host routine's sequential order (nullvec::null_vector):
// lanes only split loops whose iterations are independent (elementwise
// scaling, the trailing columns, the entries of z), so the bits agree.
constexpr int NV_WARPS = 4;
__global__ void __launch_bounds__(NV_WARPS * 32) k_null_vectors(const double* __restrict__ T, int ell,
                                                                const int32_t* __restrict__ ptr,
                                                                const int32_t* __restrict__ idx, int nsets,
                                                                double* __restrict__ Z, double* __restrict__ res) {
  using namespace nullvec;
  constexpr int ME = MAX_ELL;
  __shared__ double Ash[NV_WARPS][ME * ME];
  __shared__ double zsh[NV_WARPS][ME], tsh[NV_WARPS][ME], wsh[NV_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * NV_WARPS + warp;
  if (s >= nsets) return;
  double* A = Ash[warp];
  double* z = zsh[warp];
  double* tau = tsh[warp];
  const int r0 = ptr[s], sz = ptr[s + 1] - r0;
  double* zo = Z + (int64_t)s * ell;
  if (sz >= ell) {   // no null vector (the host planner raises DegenerateTagsError)
    for (int i = lane; i < ell; i += 32) zo[i] = 0.0;
    if (lane == 0) res[s] = INFINITY;
    return;
  }
  for (int e = lane; e < ell * sz; e += 32) {
    const int j = e / ell, i = e - j * ell;
    A[i + j * ell] = T[(int64_t)idx[r0 + j] * ell + i];
  }
  for (int j = lane; j < sz; j += 32) tau[j] = 0.0;
  __syncwarp();
  for (int j = 0; j < sz; ++j) {
    double* col = &A[j * ell];
    double inv = 0.0, beta = 0.0;
    bool skip = false;
    if (lane == 0) {
      const double alpha = col[j];
      double ss = 0.0, scale = 0.0;
      for (int i = j + 1; i < ell; ++i) scale = fmax(scale, fabs(col[i]));
      if (scale > 0.0) {
        const double inv_scale = div(1.0, scale);
        for (int i = j + 1; i < ell; ++i) {
          const double x = mul(col[i], inv_scale);
          ss = add(ss, mul(x, x));
        }
      }
      const double xnorm = mul(scale, sqrt_(ss));
      if (xnorm == 0.0) {
        skip = true;
      } else {
        const double aa = fabs(alpha), wmax = fmax(aa, xnorm), zmin = fmin(aa, xnorm);
        const double ratio = div(zmin, wmax);
        beta = -copysign(mul(wmax, sqrt_(add(1.0, mul(ratio, ratio)))), alpha);
        tau[j] = div(sub(beta, alpha), beta);
        inv = div(1.0, sub(alpha, beta));
      }
    }
    skip = __shfl_sync(0xffffffffu, skip, 0);
    if (skip) continue;   // tau_j = 0, column untouched
    inv = __shfl_sync(0xffffffffu, inv, 0);
    beta = __shfl_sync(0xffffffffu, beta, 0);
    for (int i = j + 1 + lane; i < ell; i += 32) col[i] = mul(col[i], inv);
    __syncwarp();
    if (lane == 0) col[j] = beta;
    const double tj = tau[j];
    for (int c = j + 1 + lane; c < sz; c += 32) {   // trailing columns, one lane each
      double* a = &A[c * ell];
      double w = a[j];
      for (int i = j + 1; i < ell; ++i) w = add(w, mul(col[i], a[i]));
      w = mul(w, tj);
      a[j] = sub(a[j], w);
      for (int i = j + 1; i < ell; ++i) a[i] = sub(a[i], mul(w, col[i]));
    }
    __syncwarp();
  }
  for (int i = lane; i < ell; i += 32) z[i] = (i == ell - 1) ? 1.0 : 0.0;
  __syncwarp();
  for (int j = sz - 1; j >= 0; --j) {
    const double* v = &A[j * ell];
    if (lane == 0) {
      double w = z[j];
      for (int i = j + 1; i < ell; ++i) w = add(w, mul(v[i], z[i]));
      wsh[warp] = mul(w, tau[j]);
    }
    __syncwarp();
    const double w = wsh[warp];
    if (lane == 0) z[j] = sub(z[j], w);
    for (int i = j + 1 + lane; i < ell; i += 32) z[i] = sub(z[i], mul(w, v[i]));
    __syncwarp();
  }
  // residual ||T[rows] z||: per-row dots by lanes, sum of squares in order by lane 0
  double* d = tau;   // reuse
  for (int j = lane; j < sz; j += 32) {
    const double* t = T + (int64_t)idx[r0 + j] * ell;
    double dd = 0.0;
    for (int i = 0; i < ell; ++i) dd = add(dd, mul(t[i], z[i]));
    d[j] = dd;
  }
  __syncwarp();
  if (lane == 0) {
    double r2 = 0.0;
    for (int j = 0; j < sz; ++j) r2 = add(r2, mul(d[j], d[j]));
    res[s] = sqrt_(r2);
  }
  for (int i = lane; i < ell; i += 32) zo[i] = z[i];
}
}  // namespace
}  // namespace ublr

extern "C" int ublr_null_vectors_device(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int nsets,
                                        double* Z, double* res, void* stream) {
  UBLR_REQUIRE(T && ell >= 1 && ell <= ublr::nullvec::MAX_ELL && ptr && idx && nsets >= 0 && Z && res,
               UBLR_ERR_VALUE, "ublr_null_vectors_device: bad arguments (ell <= 32)");
  if (nsets == 0) return UBLR_OK;
  ublr::k_null_vectors<<<(nsets + ublr::NV_WARPS - 1) / ublr::NV_WARPS, ublr::NV_WARPS * 32, 0, (cudaStream_t)stream>>>(T, ell, ptr, idx, nsets, Z, res);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
