// K6 + K7 fused for small blocks (m_max <= 64, k <= 32: configs 1 and 2).
//
// direct_core (ref/reconstruction.py:185-198) needs C_ij = U_i^T A_ij V_j for
// every block pair; structured_identity_discrepancy (ref/reconstruction.py:
// 201-244, colour-probe semantics incl. the same-colour leak)
// needs, for each near pair p = (i, j*),
//   B_p[:, q] = sum_{j' in colour(j*), q < m_j'} (A_ij' - U_i C_ij' V_j'^T)[:, q].
// Both read the same operator entries A_ij' and the second needs exactly the
// C_ij' of the first, so one CTA per (block row i, colour c) walks the
// members j of colour c once:
//   generate A_ij (thread = one column q, 16 rows) into shared memory and,
//     if block row i has a near pair of colour c, add it to D (registers);
//   T = U_i^T A_ij            (KP x 64, DMMA, warp = 8 columns q)
//   C_ij = T V_j              (KP x KP, DMMA) -> core
//   S += C_ij V_j^T           (KP x 64, DMMA, accumulators live across j)
// and finally B_p = D - U_i S. The operator is evaluated once per entry
// instead of twice (coupling + probe), and the S workspace, the per-pair
// probe kernels and their launches disappear. Entries are the same bits as
// the other kernels' (kernel_entry: squared distance of the coordinate
// differences, diagonal from op.diag).
#include "common.cuh"
#include "optile.cuh"

namespace ublr {
namespace {

constexpr int CS_THREADS = 256;
constexpr int CS_M = 64;           // block size bound
constexpr int CS_SA = CS_M + 4;    // A / T row stride (doubles)

template <int KP>
struct CsLayout {
  static constexpr int SU = KP + 4;   // U_i, V_j rows
  static constexpr int SC = KP + 4;   // C_ij rows
  static constexpr int A = 0;                       // [64][SA]   A_ij (r, q)
  static constexpr int U = A + CS_M * CS_SA;        // [64][SU]   U_i (r, a)
  static constexpr int V = U + CS_M * SU;           // [64][SU]   V_j (q, c)
  static constexpr int T = V + CS_M * SU;           // [KP][SA]   T (a, q); S at the end
  static constexpr int C = T + KP * CS_SA;          // [KP][SC]
  static constexpr int X = C + KP * SC;             // [3][64]    row coordinates of block i
  static constexpr int TOTAL = X + 3 * CS_M;
  static constexpr size_t bytes() { return (size_t)TOTAL * sizeof(double); }
};

template <int KIND, int KP>
__global__ void __launch_bounds__(CS_THREADS) k_coupling_nf_small(
    ublr_op_t op, const int32_t* __restrict__ off, const int32_t* __restrict__ roff, const double* __restrict__ U,
    const double* __restrict__ V, int64_t lduv, double* __restrict__ core, int64_t ldc,
    const int32_t* __restrict__ cptr, const int32_t* __restrict__ cidx, int n_colours,
    const int32_t* __restrict__ pair_of, const int32_t* __restrict__ nidx, const int64_t* __restrict__ b_off,
    double* __restrict__ B, int i0) {
  using L = CsLayout<KP>;
  constexpr int SU = L::SU, SC = L::SC, NA = KP / 8;
  __shared__ LogTables lt;
  extern __shared__ double dsm[];
  double* As = dsm + L::A;
  double* Us = dsm + L::U;
  double* Vs = dsm + L::V;
  double* Ts = dsm + L::T;
  double* Cs = dsm + L::C;
  double* xr = dsm + L::X;
  const int i = i0 + blockIdx.x, c = blockIdx.y;
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int ki = roff[i + 1] - roff[i];
  const int p = pair_of[(int64_t)i * n_colours + c];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  // U_i (zero-padded to 64 x KP) and the row points of block i
  for (int e = tid; e < CS_M * KP; e += CS_THREADS) {
    const int r = e / KP, a = e - r * KP;
    Us[r * SU + a] = (r < mi && a < ki) ? U[(int64_t)(ri0 + r) * lduv + a] : 0.0;
  }
  if (tid < CS_M) {
    const int r = tid;
    if (KIND == UBLR_OP_DENSE) {
      xr[r] = (r < mi) ? (double)(op.perm ? op.perm[ri0 + r] : ri0 + r) : 0.0;
    } else {
      for (int a = 0; a < 3; ++a) xr[a * CS_M + r] = (r < mi && a < op.dim) ? op.coords[(int64_t)a * op.n + ri0 + r] : 0.0;
    }
  }
  // generation role: column q, rows r0 + 4 s
  const int q = tid & (CS_M - 1), r0 = tid >> 6;
  double D[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) D[s] = 0.0;
  // S accumulators: warp owns columns 8 warp .. 8 warp + 7, all KP rows
  double S[NA][2];
#pragma unroll
  for (int a = 0; a < NA; ++a) S[a][0] = S[a][1] = 0.0;
  const bool near = p >= 0;
  __syncthreads();

  const int mem0 = cptr[c], mem1 = cptr[c + 1];
  // the column point of the first member; later ones are loaded one member ahead
  RowPoint cp_next;
  {
    const int j = cidx[mem0];
    cp_next = load_row_point(op, off[j] + q, q < off[j + 1] - off[j]);
  }
  for (int mem = mem0; mem < mem1; ++mem) {
    const int j = cidx[mem];
    const int cj0 = off[j], mj = off[j + 1] - cj0;
    const int kj = roff[j + 1] - roff[j];
    // ---- V_j -> shared (cp.async, zero-filled padding), overlapping the generation
    for (int e = tid; e < CS_M * KP; e += CS_THREADS) {
      const int r = e / KP, a = e - r * KP;
      const bool ok = r < mj && a < kj;
      cp_async8(&Vs[r * SU + a], ok ? (const void*)(V + (int64_t)(cj0 + r) * lduv + a) : (const void*)V, ok);
    }
    cp_async_commit();
    // ---- A_ij -> shared (and D)
    {
      const bool qok = q < mj;
      const RowPoint cp = cp_next;   // the column point
      if (mem + 1 < mem1) {
        const int jn = cidx[mem + 1];
        cp_next = load_row_point(op, off[jn] + q, q < off[jn + 1] - off[jn]);
      }
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const int r = r0 + 4 * s;
        double v = 0.0;
        if (qok && r < mi) {
          if (KIND == UBLR_OP_DENSE) {
            const int orow = (int)xr[r];
            v = op.transpose ? op.A[(int64_t)cp.orig * op.lda + orow] : op.A[(int64_t)orow * op.lda + cp.orig];
          } else {
            v = kernel_entry<KIND>(op, cp, ri0 + r, xr[r], xr[CS_M + r], xr[2 * CS_M + r], &lt);
          }
        }
        As[r * CS_SA + q] = v;
        D[s] += v;
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---- T = U_i^T A_ij: warp owns columns q0 = 8 warp, all KP rows; K = 64 rows r
    {
      const int q0 = warp * 8;
      double acc[NA][2];
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a][0] = acc[a][1] = 0.0;
#pragma unroll 4
      for (int k4 = 0; k4 < CS_M; k4 += 4) {
        const double bv = As[(k4 + t) * CS_SA + q0 + g];
#pragma unroll
        for (int a = 0; a < NA; ++a) mma8x8x4(acc[a][0], acc[a][1], Us[(k4 + t) * SU + a * 8 + g], bv);
      }
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        Ts[(a * 8 + g) * CS_SA + q0 + 2 * t] = acc[a][0];
        Ts[(a * 8 + g) * CS_SA + q0 + 2 * t + 1] = acc[a][1];
      }
    }
    __syncthreads();
    // ---- C_ij = T V_j: NA x NA tiles over the warps; K = 64 columns q
    for (int tile = warp; tile < NA * NA; tile += CS_THREADS / 32) {
      const int ta = tile / NA, tc = tile - ta * NA;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
      for (int k4 = 0; k4 < CS_M; k4 += 4)
        mma8x8x4(c0, c1, Ts[(ta * 8 + g) * CS_SA + k4 + t], Vs[(k4 + t) * SU + tc * 8 + g]);
      const int a = ta * 8 + g, cc = tc * 8 + 2 * t;
      Cs[a * SC + cc] = c0;
      Cs[a * SC + cc + 1] = c1;
      if (a < ki) {
        double* dst = core + (int64_t)(roff[i] + a) * ldc + roff[j];
        if (cc < kj) dst[cc] = c0;
        if (cc + 1 < kj) dst[cc + 1] = c1;
      }
    }
    __syncthreads();
    // ---- S += C_ij V_j^T: warp owns columns q0 = 8 warp; K = KP
    if (near) {
      const int q0 = warp * 8;
#pragma unroll
      for (int k4 = 0; k4 < KP; k4 += 4) {
        const double bv = Vs[(q0 + g) * SU + k4 + t];
#pragma unroll
        for (int a = 0; a < NA; ++a) mma8x8x4(S[a][0], S[a][1], Cs[(a * 8 + g) * SC + k4 + t], bv);
      }
    }
    __syncthreads();   // As, Vs, Ts, Cs are rewritten by the next member
  }
  if (!near) return;
  // ---- B_p = D - U_i S for the near pair p = (i, j*), columns q < m_j*
  double* Ss = Ts;
  {
    const int q0 = warp * 8;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      Ss[(a * 8 + g) * CS_SA + q0 + 2 * t] = S[a][0];
      Ss[(a * 8 + g) * CS_SA + q0 + 2 * t + 1] = S[a][1];
    }
  }
  __syncthreads();
  // U_i S (64 x 64) by DMMA: warp w owns rows 8w .. 8w + 7; the padding
  // columns of U_i and rows of S are zero, so K = KP adds exact zeros only
  double* US = As;   // free after the member loop
  {
    double acc[8][2];
#pragma unroll
    for (int qb = 0; qb < 8; ++qb) acc[qb][0] = acc[qb][1] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < KP; k4 += 4) {
      const double av = Us[(warp * 8 + g) * SU + k4 + t];
#pragma unroll
      for (int qb = 0; qb < 8; ++qb) mma8x8x4(acc[qb][0], acc[qb][1], av, Ss[(k4 + t) * CS_SA + qb * 8 + g]);
    }
#pragma unroll
    for (int qb = 0; qb < 8; ++qb) {
      US[(warp * 8 + g) * CS_SA + qb * 8 + 2 * t] = acc[qb][0];
      US[(warp * 8 + g) * CS_SA + qb * 8 + 2 * t + 1] = acc[qb][1];
    }
  }
  __syncthreads();
  const int jn = nidx[p];
  const int mjn = off[jn + 1] - off[jn];
  if (q >= mjn) return;
  double* Bp = B + b_off[p];
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int r = r0 + 4 * s;
    if (r < mi) Bp[(int64_t)r * mjn + q] = D[s] - US[r * CS_SA + q];
  }
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_coupling_nearfield(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                                       const double* U, const double* V, int64_t ld_uv, double* core, int64_t ld_c,
                                       const int32_t* cptr, const int32_t* cidx, int n_colours, int m_max,
                                       const int32_t* pair_of, const int32_t* nidx, const int64_t* b_off, double* B,
                                       void* stream, int i0, int i1) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && n_colours > 0 && off && roff && U && V && core && cptr && cidx && pair_of && nidx && b_off &&
                   B && k >= 1 && ld_uv >= k,
               UBLR_ERR_VALUE, "ublr_coupling_nearfield: bad arguments");
  UBLR_REQUIRE(m_max <= CS_M, UBLR_ERR_VALUE, "ublr_coupling_nearfield: supports m <= 64");
  UBLR_REQUIRE(0 <= i0 && i0 < i1 && i1 <= b && n_colours <= 65535, UBLR_ERR_VALUE,
               "ublr_coupling_nearfield: bad block-row range");
  const int kk = k < m_max ? k : m_max;
  UBLR_REQUIRE(kk <= 32, UBLR_ERR_VALUE, "ublr_coupling_nearfield: supports k <= 32");
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)(i1 - i0), (unsigned)n_colours);
#define UBLR_CS(KPv)                                                                                              \
  UBLR_DISPATCH_KIND(op->kind, KIND, {                                                                            \
    size_t sm = CsLayout<KPv>::bytes();                                                                           \
    UBLR_CUDA(cudaFuncSetAttribute(k_coupling_nf_small<KIND, KPv>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                   (int)sm));                                                                    \
    k_coupling_nf_small<KIND, KPv><<<grid, CS_THREADS, sm, st>>>(*op, off, roff, U, V, ld_uv, core, ld_c, cptr,    \
                                                                 cidx, n_colours, pair_of, nidx, b_off, B, i0);   \
  })
  if (kk <= 8) { UBLR_CS(8); }
  else if (kk <= 16) { UBLR_CS(16); }
  else if (kk <= 24) { UBLR_CS(24); }
  else { UBLR_CS(32); }
#undef UBLR_CS
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
