// K12b — exact blockwise Frobenius norms of the parity gates (BASELINE.json):
//   ublr_frob_error: per pair (i, j), ||A_ij - A_hat_ij||_F^2 and ||A_ij||_F^2,
//                    with A_ij generated on the fly from the operator
//                    descriptor (A is never materialised);
//   ublr_frob_diff:  per pair, ||A_hat1_ij - A_hat2_ij||_F^2 for two compressed
//                    representations on the same tessellation.
// A_hat_ij = U_i C_ij V_j^T (+ B_ij on near pairs) is ref/reconstruction.py:50-132
// (UniformBLR); the gates are SURVEY.md §8(d) / BASELINE.json north star.
//
// The difference is formed entry by entry (the algebraic shortcut
// ||A||^2 - 2<A, A_hat> + ||C||^2 cancels catastrophically at 1e-13
// relative). One CTA per pair; the pair is swept in 64 x 64 tiles:
//   W = [-C1_ij V1_j^T ; +C2_ij V2_j^T]  (k1 + k2) x 64   (shared memory)
//   D = M + [U1_i | U2_i] W - B1_ij                          (4 x 4 per thread)
// with M = A_ij (error) or B2_ij (difference). Per-pair sums are reduced in a
// fixed order (warp shuffles, then warp partials in order): the result is
// deterministic. Work per pair 2 m_i m_j (k1 + k2) + 2 (k1 + k2) k m_j flops.
#include "optile.cuh"

namespace ublr {
namespace {

constexpr int FT = 256;   // threads
constexpr int TQ = 64;    // columns per tile
constexpr int TR = 64;    // rows per slab
constexpr int FK_MAX = 96;  // k1 + k2

struct Rep {
  const double* U;
  const double* V;
  int64_t ld_uv;
  const double* core;
  int64_t ld_c;
  const int32_t* roff;
  const double* B;
};

template <int KIND, int MODE>
__global__ void __launch_bounds__(FT) k_frob(ublr_op_t op, Rep r1, Rep r2, int k1max, int k2max,
                                             const int32_t* __restrict__ off, const int32_t* __restrict__ nptr,
                                             const int32_t* __restrict__ nidx, const int64_t* __restrict__ b_off,
                                             int b, int i0, double* __restrict__ err2, double* __restrict__ a2) {
  extern __shared__ double sm[];
  const int j = blockIdx.x, i = i0 + blockIdx.y;
  const int tid = threadIdx.x;
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int cj0 = off[j], mj = off[j + 1] - cj0;
  const int k1i = r1.roff[i + 1] - r1.roff[i], k1j = r1.roff[j + 1] - r1.roff[j];
  const int k2i = MODE == 1 ? r2.roff[i + 1] - r2.roff[i] : 0;
  const int k2j = MODE == 1 ? r2.roff[j + 1] - r2.roff[j] : 0;
  const int KC = k1i + k2i;
  const int LDU = k1max + k2max + 1;
  int pnear = -1;
  for (int q = nptr[i]; q < nptr[i + 1]; ++q)
    if (nidx[q] == j) pnear = q;

  double* sC1 = sm;                                  // k1max x k1max
  double* sC2 = sC1 + k1max * k1max;                 // k2max x k2max
  double* sV1 = sC2 + k2max * k2max;                 // TQ x k1max
  double* sV2 = sV1 + TQ * k1max;                    // TQ x k2max
  double* sW = sV2 + TQ * k2max;                     // (k1max + k2max) x TQ
  double* sU = sW + (k1max + k2max) * TQ;            // TR x LDU
  double* red = sU + TR * LDU;                       // 2 x 8 warp partials
  LogTables* lt = reinterpret_cast<LogTables*>(red + 16);
  if (KIND == UBLR_OP_LOG) init_log_tables(lt);

  for (int e = tid; e < k1i * k1j; e += FT) {
    int a = e / k1j, c = e - a * k1j;
    sC1[a * k1max + c] = r1.core[(int64_t)(r1.roff[i] + a) * r1.ld_c + r1.roff[j] + c];
  }
  if (MODE == 1)
    for (int e = tid; e < k2i * k2j; e += FT) {
      int a = e / k2j, c = e - a * k2j;
      sC2[a * k2max + c] = r2.core[(int64_t)(r2.roff[i] + a) * r2.ld_c + r2.roff[j] + c];
    }

  const int tx = tid & 15, ty = tid >> 4;   // 4 columns x 4 rows per thread
  double e_acc = 0.0, a_acc = 0.0;
  const double* B1p = (r1.B && pnear >= 0) ? r1.B + b_off[pnear] : nullptr;
  const double* B2p = (MODE == 1 && r2.B && pnear >= 0) ? r2.B + b_off[pnear] : nullptr;

  for (int q0 = 0; q0 < mj; q0 += TQ) {
    __syncthreads();   // previous tile's sW / sU reads done (and sC loaded)
    for (int e = tid; e < TQ * k1j; e += FT) {
      int t = e / k1j, c = e - t * k1j;
      sV1[t * k1max + c] = q0 + t < mj ? r1.V[(int64_t)(cj0 + q0 + t) * r1.ld_uv + c] : 0.0;
    }
    if (MODE == 1)
      for (int e = tid; e < TQ * k2j; e += FT) {
        int t = e / k2j, c = e - t * k2j;
        sV2[t * k2max + c] = q0 + t < mj ? r2.V[(int64_t)(cj0 + q0 + t) * r2.ld_uv + c] : 0.0;
      }
    __syncthreads();
    // W rows: -C1 V1^T (a < k1i), +C2 V2^T (k1i <= a < KC)
    for (int e = tid; e < KC * TQ; e += FT) {
      int a = e / TQ, t = e - a * TQ;
      double s = 0.0;
      if (a < k1i) {
        for (int c = 0; c < k1j; ++c) s = fma(sC1[a * k1max + c], sV1[t * k1max + c], s);
        s = -s;
      } else {
        const int a2_ = a - k1i;
        for (int c = 0; c < k2j; ++c) s = fma(sC2[a2_ * k2max + c], sV2[t * k2max + c], s);
      }
      sW[a * TQ + t] = s;
    }
    for (int r0 = 0; r0 < mi; r0 += TR) {
      __syncthreads();   // sW complete; previous slab's sU reads done
      for (int e = tid; e < TR * KC; e += FT) {
        int r = e / KC, c = e - r * KC;
        double u = 0.0;
        if (r0 + r < mi) u = c < k1i ? r1.U[(int64_t)(ri0 + r0 + r) * r1.ld_uv + c]
                                     : r2.U[(int64_t)(ri0 + r0 + r) * r2.ld_uv + (c - k1i)];
        sU[r * LDU + c] = u;
      }
      __syncthreads();
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      for (int c = 0; c < KC; ++c) {
        double u[4], w[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) u[a] = sU[(4 * ty + a) * LDU + c];
#pragma unroll
        for (int t = 0; t < 4; ++t) w[t] = sW[c * TQ + 4 * tx + t];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[a][t] = fma(u[a], w[t], acc[a][t]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = r0 + 4 * ty + a;
        if (r >= mi) continue;
        RowPoint rp;
        if (MODE == 0) rp = load_row_point(op, ri0 + r, true);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int q = q0 + 4 * tx + t;
          if (q >= mj) continue;
          double v = acc[a][t];
          if (MODE == 0) {
            const double av = op_entry<KIND>(op, rp, cj0 + q, lt);
            a_acc = fma(av, av, a_acc);
            v += av;
          } else if (B2p) {
            v += B2p[(int64_t)r * mj + q];
          }
          if (B1p) v -= B1p[(int64_t)r * mj + q];
          e_acc = fma(v, v, e_acc);
        }
      }
    }
  }
  // deterministic CTA reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
    a_acc += __shfl_xor_sync(0xffffffffu, a_acc, o);
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    red[tid >> 5] = e_acc;
    red[8 + (tid >> 5)] = a_acc;
  }
  __syncthreads();
  if (tid == 0) {
    double se = 0.0, sa = 0.0;
    for (int w = 0; w < FT / 32; ++w) {
      se += red[w];
      sa += red[8 + w];
    }
    const int64_t o = (int64_t)blockIdx.y * b + j;
    err2[o] = se;
    if (a2) a2[o] = sa;
  }
}

size_t frob_smem(int k1, int k2) {
  size_t d = (size_t)k1 * k1 + (size_t)k2 * k2 + (size_t)TQ * (k1 + k2) + (size_t)(k1 + k2) * TQ +
             (size_t)TR * (k1 + k2 + 1) + 16;
  return d * sizeof(double) + sizeof(LogTables);
}

template <int KIND, int MODE>
int launch_frob(const ublr_op_t& op, const Rep& r1, const Rep& r2, int k1, int k2, const int32_t* off,
                const int32_t* nptr, const int32_t* nidx, const int64_t* b_off, int b, int i0, int i1, double* err2,
                double* a2, cudaStream_t st) {
  const size_t smem = frob_smem(k1, k2);
  auto kern = k_frob<KIND, MODE>;
  UBLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int c0 = i0; c0 < i1; c0 += 65535) {   // grid.y limit
    const int c1 = c0 + 65535 < i1 ? c0 + 65535 : i1;
    dim3 grid(b, c1 - c0);
    kern<<<grid, FT, smem, st>>>(op, r1, r2, k1, k2, off, nptr, nidx, b_off, b, c0, err2 + (int64_t)(c0 - i0) * b,
                                 a2 ? a2 + (int64_t)(c0 - i0) * b : nullptr);
    UBLR_LAUNCH_CHECK();
  }
  return UBLR_OK;
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_frob_error(const ublr_op_t* op, const int32_t* off, const int32_t* nptr, const int32_t* nidx,
                               const int64_t* b_off, int b, const int32_t* roff, int k, const double* U,
                               const double* V, int64_t ld_uv, const double* core, int64_t ld_c, const double* B,
                               int i0, int i1, double* err2, double* a2, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(off && nptr && nidx && b_off && roff && b > 0 && 0 <= i0 && i0 <= i1 && i1 <= b && err2 && k >= 0 &&
                   k <= FK_MAX && (k == 0 || (U && V && core)) && ld_uv >= k,
               UBLR_ERR_VALUE, "ublr_frob_error: bad arguments (rank must be <= 96)");
  if (i1 == i0) return UBLR_OK;
  Rep r1{U, V, ld_uv, core, ld_c, roff, B};
  Rep r2{nullptr, nullptr, 0, nullptr, 0, roff, nullptr};
  cudaStream_t st = (cudaStream_t)stream;
  UBLR_DISPATCH_KIND(op->kind, KIND,
                     return launch_frob<KIND, 0>(*op, r1, r2, k, 0, off, nptr, nidx, b_off, b, i0, i1, err2, a2, st));
  return UBLR_OK;
}

extern "C" int ublr_frob_diff(const int32_t* off, const int32_t* nptr, const int32_t* nidx, const int64_t* b_off,
                              int b, const int32_t* roff1, int k1, const double* U1, const double* V1, int64_t ld1,
                              const double* core1, int64_t ldc1, const double* B1, const int32_t* roff2, int k2,
                              const double* U2, const double* V2, int64_t ld2, const double* core2, int64_t ldc2,
                              const double* B2, int i0, int i1, double* diff2, void* stream) {
  UBLR_REQUIRE(off && nptr && nidx && b_off && roff1 && roff2 && b > 0 && 0 <= i0 && i0 <= i1 && i1 <= b && diff2 &&
                   k1 >= 0 && k2 >= 0 && k1 + k2 <= FK_MAX && (k1 == 0 || (U1 && V1 && core1)) &&
                   (k2 == 0 || (U2 && V2 && core2)) && ld1 >= k1 && ld2 >= k2,
               UBLR_ERR_VALUE, "ublr_frob_diff: bad arguments (k1 + k2 must be <= 96)");
  if (i1 == i0) return UBLR_OK;
  Rep r1{U1, V1, ld1, core1, ldc1, roff1, B1};
  Rep r2{U2, V2, ld2, core2, ldc2, roff2, B2};
  ublr_op_t op{};
  op.kind = UBLR_OP_DENSE;
  return launch_frob<UBLR_OP_DENSE, 1>(op, r1, r2, k1, k2, off, nptr, nidx, b_off, b, i0, i1, diff2, nullptr,
                                       (cudaStream_t)stream);
}
