// K12 — products with the compressed representation (ref/reconstruction.py:93-119).
//
// A_hat X = U (C (V^T X)) + B X blockwise, and the adjoint
// A_hat^T X = V (C^T (U^T X)) + B^T X. Used by relative_error (the
// reference's power-method estimate, ref/reconstruction.py:160-177) and by
// parity checks; ragged blocks are supported. The K x K core product reuses
// the operator-apply GEMM (ublr_apply with a dense descriptor).
#include "common.cuh"

namespace ublr {
namespace {

constexpr int BT = 256;

// P[roff_i + a, c] = sum_r L[off_i + r, a] X[off_i + r, c]   (L = V, or U for the adjoint)
__global__ void __launch_bounds__(BT) k_blr_project(const double* __restrict__ L, int64_t ldl,
                                                    const double* __restrict__ X, int64_t ldx, int w,
                                                    const int32_t* __restrict__ off,
                                                    const int32_t* __restrict__ roff, double* __restrict__ P,
                                                    int64_t ldp) {
  const int i = blockIdx.x;
  const int r0 = off[i], m = off[i + 1] - r0;
  const int k0 = roff[i], ki = roff[i + 1] - k0;
  for (int e = threadIdx.x + blockIdx.y * BT; e < ki * w; e += BT * gridDim.y) {
    int a = e / w, c = e - a * w;
    double s = 0.0;
    for (int r = 0; r < m; ++r) s = fma(L[(int64_t)(r0 + r) * ldl + a], X[(int64_t)(r0 + r) * ldx + c], s);
    P[(int64_t)(k0 + a) * ldp + c] = s;
  }
}

// out[off_i + r, c] = sum_a R[off_i + r, a] CP[roff_i + a, c] + sum_j Bpair X_j
// (forward: pairs (i, j) j in N_i, block row-major m_i x m_j;
//  adjoint: pairs (j, i), i.e. B_ji^T, located through tpair).
__global__ void __launch_bounds__(BT) k_blr_expand(const double* __restrict__ R, int64_t ldr,
                                                   const double* __restrict__ CP, int64_t ldp,
                                                   const double* __restrict__ X, int64_t ldx, int w,
                                                   const int32_t* __restrict__ off,
                                                   const int32_t* __restrict__ roff,
                                                   const int32_t* __restrict__ nptr,
                                                   const int32_t* __restrict__ nidx,
                                                   const int32_t* __restrict__ tpair,
                                                   const int64_t* __restrict__ b_off,
                                                   const double* __restrict__ B, int adjoint,
                                                   double* __restrict__ out, int64_t ldo) {
  const int i = blockIdx.x;
  const int r0 = off[i], m = off[i + 1] - r0;
  const int k0 = roff[i], ki = roff[i + 1] - k0;
  for (int e = threadIdx.x + blockIdx.y * BT; e < m * w; e += BT * gridDim.y) {
    int r = e / w, c = e - r * w;
    double s = 0.0;
    for (int a = 0; a < ki; ++a) s = fma(R[(int64_t)(r0 + r) * ldr + a], CP[(int64_t)(k0 + a) * ldp + c], s);
    for (int q = nptr[i]; q < nptr[i + 1]; ++q) {
      int j = nidx[q];
      int cj0 = off[j], mj = off[j + 1] - cj0;
      if (!adjoint) {
        const double* Bp = B + b_off[q] + (int64_t)r * mj;          // B_ij row r
        for (int t = 0; t < mj; ++t) s = fma(Bp[t], X[(int64_t)(cj0 + t) * ldx + c], s);
      } else {
        int p = tpair[q];                                            // pair (j, i)
        const double* Bp = B + b_off[p] + r;                         // B_ji column r (m_j x m_i)
        for (int t = 0; t < mj; ++t) s = fma(Bp[(int64_t)t * m], X[(int64_t)(cj0 + t) * ldx + c], s);
      }
    }
    out[(int64_t)(r0 + r) * ldo + c] = s;
  }
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_blr_apply(const double* U, const double* V, int64_t ld_uv, const double* core, int64_t K,
                              const double* B, const int64_t* b_off, const int32_t* off, const int32_t* roff,
                              const int32_t* nptr, const int32_t* nidx, const int32_t* tpair, int b,
                              const double* X, int64_t ld_x, int w, int adjoint, double* out, int64_t ld_o,
                              double* work, void* stream) {
  UBLR_REQUIRE(U && V && B && b_off && off && roff && nptr && nidx && tpair && X && out && work && b > 0 && w >= 0,
               UBLR_ERR_VALUE, "ublr_blr_apply: bad arguments");
  if (w == 0) return UBLR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  double* P = work;           // K x w
  double* CP = work + K * w;  // K x w
  const double* L = adjoint ? U : V;
  const double* R = adjoint ? V : U;
  dim3 g1(b, 1);
  k_blr_project<<<g1, BT, 0, st>>>(L, ld_uv, X, ld_x, w, off, roff, P, w);
  UBLR_LAUNCH_CHECK();
  if (K > 0) {
    ublr_op_t op{};
    op.kind = UBLR_OP_DENSE;
    op.transpose = adjoint ? 1 : 0;
    op.A = core;
    op.lda = K;
    op.n = K;
    op.perm = nullptr;  // identity
    int rc = ublr_apply(&op, P, w, w, CP, w, stream);
    if (rc) return rc;
  }
  k_blr_expand<<<g1, BT, 0, st>>>(R, ld_uv, CP, w, X, ld_x, w, off, roff, nptr, nidx, tpair, b_off, B, adjoint,
                                  out, ld_o);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int64_t ublr_blr_apply_workspace_bytes(int64_t K, int w) {
  return (2 * K * (int64_t)w) * (int64_t)sizeof(double) + 256;
}
