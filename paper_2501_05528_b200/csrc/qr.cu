// K4 — per-block combine + Householder QR -> explicit leading Q columns.
//
// Replaces, per block i, `_combined_sample` (ref/bases.py:207-210) and
// `_basis_or_identity` / `col_basis` (ref/bases.py:78-83, ref/linalg.py:55-69):
// numpy.linalg.qr = LAPACK dgeqrf + dorgqr, i.e. Householder reflectors in the
// dlarfg convention (beta = -sign(alpha) * ||x||, v(1) = 1,
// tau = (beta - alpha) / beta) and Q = H_1 ... H_k [I; 0]. Only the first k
// sample columns are formed: Q[:, :k] of an unpivoted QR does not depend on
// later columns.
//
// One CTA per block; the m x k sample lives in shared memory (odd leading
// dimension: conflict-free column walks); each warp owns whole columns, so
// dot products are warp-shuffle reductions and a step needs two barriers.
#include "common.cuh"

namespace ublr {
namespace {

constexpr int QR_THREADS = 256;
constexpr int QR_WARPS = QR_THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(QR_THREADS) k_block_qr(const double* __restrict__ Y, int64_t ldy, int mode,
                                                         const double* __restrict__ z, int ell, int gc,
                                                         const int32_t* __restrict__ col0,
                                                         const int32_t* __restrict__ off, int k,
                                                         double* __restrict__ U, int64_t ldu,
                                                         const double* __restrict__ Y2, double* __restrict__ U2) {
  extern __shared__ double smem[];
  const int i = blockIdx.x;
  if (blockIdx.y == 1) {  // second side of a pair launch (Z -> V)
    Y = Y2;
    U = U2;
  }
  const int r0 = off[i];
  const int m = off[i + 1] - r0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* out = U + (int64_t)r0 * ldu;

  const bool plain_qr = (mode & 2) != 0;  // col_basis semantics: no identity shortcut
  mode &= 1;
  if (k >= m && !plain_qr) {  // tiny block: identity basis (ref/bases.py:80-82)
    for (int e = tid; e < m * m; e += QR_THREADS) {
      int r = e / m, c = e - r * m;
      out[(int64_t)r * ldu + c] = (r == c) ? 1.0 : 0.0;
    }
    return;
  }
  const int lds = k | 1;
  double* S = smem;                 // m x lds
  double* tau = smem + m * lds;     // k

  // 1. sample
  if (mode == 0) {
    const double* zi = z + (int64_t)i * ell;
    for (int e = tid; e < m * k; e += QR_THREADS) {
      int r = e / k, q = e - r * k;
      const double* yr = Y + (int64_t)(r0 + r) * ldy + q;
      double s = 0.0;
      for (int c = 0; c < ell; ++c) s = fma(zi[c], yr[(int64_t)c * gc], s);
      S[r * lds + q] = s;
    }
  } else {
    const int c0 = col0[i];
    for (int e = tid; e < m * k; e += QR_THREADS) {
      int r = e / k, q = e - r * k;
      S[r * lds + q] = Y[(int64_t)(r0 + r) * ldy + c0 + q];
    }
  }
  __syncthreads();

  // 2. dgeqr2 with look-ahead: warp 0 owns column j + 1 of step j's trailing
  // update (c = j + 1 + warp), so it forms reflector j + 1 right after
  // updating that column; one barrier per step.
  double* vbuf = tau + k;                // dorg2r: two reflector copies of m doubles
  auto reflector = [&](int j) {          // warp 0: dlarfg on column j (rows j..m-1)
    double ss = 0.0;
    for (int r = j + 1 + lane; r < m; r += 32) {
      double x = S[r * lds + j];
      ss = fma(x, x, ss);
    }
    ss = warp_sum(ss);
    double alpha = S[j * lds + j];
    double beta, t, scal;
    if (ss == 0.0) {
      t = 0.0; beta = alpha; scal = 1.0;
    } else {
      double nrm = sqrt(fma(alpha, alpha, ss));
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int r = j + 1 + lane; r < m; r += 32) S[r * lds + j] *= scal;
    if (lane == 0) { tau[j] = t; S[j * lds + j] = beta; }
  };
  if (warp == 0) reflector(0);
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double tj = tau[j];
    // trailing columns c > j: w = v^T S(:, c); S(:, c) -= tj * v * w (v = [1; S(j+1:, j)])
    for (int c = j + 1 + warp; c < k; c += QR_WARPS) {
      double w = (lane == 0) ? S[j * lds + c] : 0.0;
      for (int r = j + 1 + lane; r < m; r += 32) w = fma(S[r * lds + j], S[r * lds + c], w);
      w = warp_sum(w) * tj;
      if (lane == 0) S[j * lds + c] -= w;
      for (int r = j + 1 + lane; r < m; r += 32) S[r * lds + c] = fma(-w, S[r * lds + j], S[r * lds + c]);
      if (c == j + 1) {                  // warp 0: the next pivot column is final
        __syncwarp();
        reflector(j + 1);
      }
    }
    __syncthreads();
  }

  // 3. dorg2r: Q = H_0 ... H_{k-1} [I; 0], in place, right to left. v_j is
  // read from a copy (vbuf, double-buffered) so that column j can be formed
  // in the same step as the update of columns c > j: one barrier per step.
  const int fw = QR_WARPS - 1;           // the warp that forms columns and stages reflectors
  if (warp == fw)
    for (int r = lane; r < m; r += 32) vbuf[((k - 1) & 1) * m + r] = r > k - 1 ? S[r * lds + k - 1] : 0.0;
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double tj = tau[j];
    const double* v = vbuf + (j & 1) * m;   // v_j below the diagonal (v_j[j] = 1 implicit)
    for (int c = j + 1 + warp; c < k; c += QR_WARPS) {
      // column c of the partially formed Q: apply H_j (rows < c of column c are zero)
      double w = (lane == 0) ? S[j * lds + c] : 0.0;
      for (int r = j + 1 + lane; r < m; r += 32) w = fma(v[r], S[r * lds + c], w);
      w = warp_sum(w) * tj;
      if (lane == 0) S[j * lds + c] -= w;
      for (int r = j + 1 + lane; r < m; r += 32) S[r * lds + c] = fma(-w, v[r], S[r * lds + c]);
    }
    if (warp == fw) {
      // column j itself: e_j - tau v; and stage v_{j-1} for the next step
      for (int r = lane; r < m; r += 32) {
        double x;
        if (r < j) x = 0.0;
        else if (r == j) x = 1.0 - tj;
        else x = -tj * v[r];
        S[r * lds + j] = x;
        if (j > 0) vbuf[((j - 1) & 1) * m + r] = r > j - 1 ? S[r * lds + j - 1] : 0.0;
      }
    }
    __syncthreads();
  }

  // 4. write U_i (m x k)
  for (int e = tid; e < m * k; e += QR_THREADS) {
    int r = e / k, q = e - r * k;
    out[(int64_t)r * ldu + q] = S[r * lds + q];
  }
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_block_qr(const double* Y, int64_t ld_y, int mode, const double* z, int ell, int gc,
                             const int32_t* col0, const int32_t* off, int b, int k, double* U, int64_t ld_u,
                             void* stream, int m_max) {
  UBLR_REQUIRE(b > 0 && off && U && Y && k >= 1 && m_max >= 1, UBLR_ERR_VALUE, "ublr_block_qr: bad arguments");
  UBLR_REQUIRE(mode >= 0 && mode <= 3, UBLR_ERR_VALUE, "ublr_block_qr: mode must be 0/1 (+2: plain QR)");
  UBLR_REQUIRE((mode & 1) || (z && ell >= 1 && gc >= k), UBLR_ERR_VALUE, "ublr_block_qr: tag mode needs z, ell, gc >= k");
  UBLR_REQUIRE(!(mode & 1) || col0, UBLR_ERR_VALUE, "ublr_block_qr: cols mode needs col0");
  UBLR_REQUIRE(ld_u >= k && ld_u >= (k < m_max ? k : m_max), UBLR_ERR_VALUE, "ublr_block_qr: ld_u too small");
  int lds = k | 1;
  size_t smem = (size_t)(m_max * lds + k + 2 * m_max) * sizeof(double);
  UBLR_REQUIRE(smem <= 220 * 1024, UBLR_ERR_VALUE, "ublr_block_qr: m*k sample exceeds shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  UBLR_CUDA(cudaFuncSetAttribute(k_block_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_block_qr<<<b, QR_THREADS, smem, st>>>(Y, ld_y, mode, z, ell, gc, col0, off, k, U, ld_u, nullptr, nullptr);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_block_qr_pair(const double* Y, const double* Z, int64_t ld_y, const double* z, int ell, int gc,
                                  const int32_t* off, int b, int k, double* U, double* V, int64_t ld_u, void* stream,
                                  int m_max) {
  UBLR_REQUIRE(b > 0 && off && U && V && Y && Z && z && k >= 1 && m_max >= 1 && ell >= 1 && gc >= k,
               UBLR_ERR_VALUE, "ublr_block_qr_pair: bad arguments");
  UBLR_REQUIRE(ld_u >= k && ld_u >= (k < m_max ? k : m_max), UBLR_ERR_VALUE, "ublr_block_qr_pair: ld_u too small");
  int lds = k | 1;
  size_t smem = (size_t)(m_max * lds + k + 2 * m_max) * sizeof(double);
  UBLR_REQUIRE(smem <= 220 * 1024, UBLR_ERR_VALUE, "ublr_block_qr_pair: m*k sample exceeds shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  UBLR_CUDA(cudaFuncSetAttribute(k_block_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_block_qr<<<dim3(b, 2), QR_THREADS, smem, st>>>(Y, ld_y, 0, z, ell, gc, nullptr, off, k, U, ld_u, Z, V);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
