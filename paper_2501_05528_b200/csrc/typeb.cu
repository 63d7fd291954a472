// Type-B helpers (ref/reconstruction.py:252-421) that are not plain GEMMs.
//
// * ublr_tag_combine_pairs: per near pair p = (i, j) the tag-combined sketch
//   rows  comb_p[r, q] = sum_c w_p[c] * Y[off_i + r, c*gc + q]
//   (the `np.tensordot(groups, z)` of ref/reconstruction.py:360-362, with the
//   1/denominator folded into w_p). One CTA per (pair, row tile); Y rows are
//   read once per CTA and every output is written once (HBM-bound).
// * ublr_assemble_tagged: explicit tagged test matrix
//   Omega[r, c*gc + q] = T[block(r), c] * G[r, q] (ref/bases.py:126-137), used
//   by the least-squares core where Omega enters dense products.
#include "common.cuh"

namespace ublr {
namespace {

constexpr int CT = 256;

__global__ void __launch_bounds__(CT) k_tag_combine_pairs(const double* __restrict__ Y, int64_t ldy, int gc, int ell,
                                                          const double* __restrict__ w, const int32_t* __restrict__ pair_i,
                                                          const int32_t* __restrict__ off, int m_max,
                                                          double* __restrict__ out) {
  __shared__ double ws[32];
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int r0 = off[i], m = off[i + 1] - r0;
  if (threadIdx.x < ell) ws[threadIdx.x] = w[(int64_t)p * ell + threadIdx.x];
  __syncthreads();
  double* o = out + (int64_t)p * m_max * gc;
  for (int64_t e = (int64_t)blockIdx.y * CT + threadIdx.x; e < (int64_t)m * gc; e += (int64_t)gridDim.y * CT) {
    int r = (int)(e / gc), q = (int)(e % gc);
    const double* yr = Y + (int64_t)(r0 + r) * ldy + q;
    // the null-vector weights cancel the near-field part of every Y_c, so
    // the result is far smaller than the terms: a compensated dot product
    // (error-free products and TwoSum, errors summed apart) keeps the
    // combination's own rounding out of the near blocks -- the kernel is
    // HBM-bound, the extra FP64 operations are free
    double s = 0.0, comp = 0.0;
    for (int c = 0; c < ell; ++c) {
      const double wy = ws[c], y = yr[(int64_t)c * gc];
      const double pr = wy * y, pe = fma(wy, y, -pr);
      const double t = s + pr, bb = t - s;
      comp += ((s - (t - bb)) + (pr - bb)) + pe;
      s = t;
    }
    o[(int64_t)r * gc + q] = s + comp;
  }
}

__global__ void __launch_bounds__(CT) k_assemble_tagged(const double* __restrict__ T, int ell,
                                                        const double* __restrict__ G, int64_t ldg, int gc,
                                                        const int32_t* __restrict__ off, int b,
                                                        double* __restrict__ out, int64_t ldo, int64_t n) {
  const int64_t tot = n * (int64_t)ell * gc;
  for (int64_t e = (int64_t)blockIdx.x * CT + threadIdx.x; e < tot; e += (int64_t)gridDim.x * CT) {
    int64_t r = e / ((int64_t)ell * gc);
    int cc = (int)(e % ((int64_t)ell * gc));
    int c = cc / gc, q = cc % gc;
    // block of row r (binary search over off)
    int lo = 0, hi = b;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (off[mid] <= r) lo = mid; else hi = mid;
    }
    out[r * ldo + cc] = T[(int64_t)lo * ell + c] * G[r * ldg + q];
  }
}

// Near blocks between the flat neighbour-CSR layout (block p at b_off[p],
// m_i x m_j row-major) and a padded per-pair layout (p * m_max * m_max,
// row stride m_max) used by the batched solves of ragged tessellations.
__global__ void __launch_bounds__(CT) k_pairs_pad(double* __restrict__ flat, const int64_t* __restrict__ b_off,
                                                  const int32_t* __restrict__ pair_i, const int32_t* __restrict__ nidx,
                                                  const int32_t* __restrict__ off, int m_max,
                                                  double* __restrict__ padded, int to_padded) {
  const int p = blockIdx.x;
  const int i = pair_i[p], j = nidx[p];
  const int mi = off[i + 1] - off[i], mj = off[j + 1] - off[j];
  double* pd = padded + (int64_t)p * m_max * m_max;
  double* fl = flat + b_off[p];
  for (int e = blockIdx.y * CT + threadIdx.x; e < mi * mj; e += gridDim.y * CT) {
    const int r = e / mj, c = e - r * mj;
    if (to_padded) pd[(int64_t)r * m_max + c] = fl[e];
    else fl[e] = pd[(int64_t)r * m_max + c];
  }
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_pairs_pad(double* flat, const int64_t* b_off, const int32_t* pair_i, const int32_t* nidx,
                              const int32_t* off, int n_pairs, int m_max, double* padded, int to_padded, void* stream) {
  UBLR_REQUIRE(flat && b_off && pair_i && nidx && off && padded && n_pairs >= 0 && m_max > 0, UBLR_ERR_VALUE,
               "ublr_pairs_pad: bad arguments");
  if (!n_pairs) return UBLR_OK;
  int gy = (m_max * m_max + CT * 4 - 1) / (CT * 4);
  dim3 grid(n_pairs, gy < 1 ? 1 : gy);
  k_pairs_pad<<<grid, CT, 0, (cudaStream_t)stream>>>(flat, b_off, pair_i, nidx, off, m_max, padded, to_padded);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_tag_combine_pairs(const double* Y, int64_t ld_y, int gc, int ell, const double* w,
                                      const int32_t* pair_i, const int32_t* off, int n_pairs, int m_max, double* out,
                                      void* stream) {
  UBLR_REQUIRE(Y && w && pair_i && off && out && gc > 0 && ell > 0 && ell <= 32 && n_pairs >= 0, UBLR_ERR_VALUE,
               "ublr_tag_combine_pairs: bad arguments");
  if (!n_pairs) return UBLR_OK;
  int64_t per = (int64_t)m_max * gc;
  int gy = (int)((per + CT * 8 - 1) / (CT * 8));
  dim3 grid(n_pairs, gy < 1 ? 1 : gy);
  k_tag_combine_pairs<<<grid, CT, 0, (cudaStream_t)stream>>>(Y, ld_y, gc, ell, w, pair_i, off, m_max, out);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_assemble_tagged(const double* T, int ell, const double* G, int64_t ld_g, int gc, const int32_t* off,
                                    int b, double* out, int64_t ld_o, int64_t n, void* stream) {
  UBLR_REQUIRE(T && G && off && out && ell > 0 && gc > 0 && b > 0 && n > 0, UBLR_ERR_VALUE,
               "ublr_assemble_tagged: bad arguments");
  int64_t tot = n * ell * gc;
  int grid = (int)((tot + CT - 1) / CT < 8192 ? (tot + CT - 1) / CT : 8192);
  k_assemble_tagged<<<grid, CT, 0, (cudaStream_t)stream>>>(T, ell, G, ld_g, gc, off, b, out, ld_o, n);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
