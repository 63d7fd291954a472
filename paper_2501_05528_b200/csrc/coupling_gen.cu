// K6 / K7 for any block size and rank (type-A reconstruction,
// ref/reconstruction.py:185-244): the tuned kernels of coupling.cu cover
// m <= 256, k <= 64 (every BASELINE config); these take over beyond that
// (e.g. the paper's own N = 100k, k = 30 setting: b = 169 boxes of up to 625
// points, suggest_block_count at ref/tessellation.py:127-140).
//
// coupling: C_ij = U_i^T A_ij V_j per CTA (i, j), swept in 32-column tiles of
//   block j: T = U_i^T A_ij[:, tile] (k_i x 32, A generated on the fly in
//   64-row slabs), then C += T V_j[tile] (thread-owned accumulators).
// near field: S_p = sum_{j' in colour(j)} C_ij' V_j'^T (k_i x m, per pair) and
//   B_p[:, q] = sum_{j'} A_ij'[:, q] - U_i S_p[:, q]  (SURVEY F11 leak).
#include "optile.cuh"

namespace ublr {
namespace {

constexpr int GT = 256;
constexpr int GQ = 32;    // columns per tile
constexpr int GR = 64;    // rows per slab
constexpr int GK_MAX = 96;

template <int KIND>
__global__ void __launch_bounds__(GT) k_coupling_gen(ublr_op_t op, const int32_t* __restrict__ off,
                                                     const int32_t* __restrict__ roff, const double* __restrict__ U,
                                                     const double* __restrict__ V, int64_t lduv,
                                                     double* __restrict__ core, int64_t ldc, int i0, int kmax) {
  extern __shared__ double sm[];
  const int j = blockIdx.x, i = i0 + blockIdx.y;
  const int tid = threadIdx.x;
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int cj0 = off[j], mj = off[j + 1] - cj0;
  const int ki = roff[i + 1] - roff[i], kj = roff[j + 1] - roff[j];
  double* sA = sm;                    // GR x GQ
  double* sU = sA + GR * GQ;          // GR x (kmax + 1)
  double* sT = sU + GR * (kmax + 1);  // kmax x GQ
  double* sV = sT + kmax * GQ;        // GQ x (kmax + 1)
  LogTables* lt = reinterpret_cast<LogTables*>(sV + GQ * (kmax + 1));
  if (KIND == UBLR_OP_LOG) init_log_tables(lt);
  const int LDU = kmax + 1;
  // T ownership: column q = tid % GQ, rows a = tid / GQ + 8 s
  const int tq = tid % GQ, ta = tid / GQ;
  constexpr int TS = GK_MAX / 8;
  // C ownership: entries e = tid + GT s of the ki x kj block
  constexpr int CS = (GK_MAX * GK_MAX + GT - 1) / GT;
  double cacc[CS];
#pragma unroll
  for (int s = 0; s < CS; ++s) cacc[s] = 0.0;

  for (int q0 = 0; q0 < mj; q0 += GQ) {
    double tacc[TS];
#pragma unroll
    for (int s = 0; s < TS; ++s) tacc[s] = 0.0;
    for (int r0 = 0; r0 < mi; r0 += GR) {
      __syncthreads();
      for (int e = tid; e < GR * GQ; e += GT) {
        const int r = e / GQ, q = e - r * GQ;
        double v = 0.0;
        if (r0 + r < mi && q0 + q < mj) {
          RowPoint rp = load_row_point(op, ri0 + r0 + r, true);
          v = op_entry<KIND>(op, rp, cj0 + q0 + q, lt);
        }
        sA[e] = v;
      }
      for (int e = tid; e < GR * ki; e += GT) {
        const int r = e / ki, a = e - r * ki;
        sU[r * LDU + a] = r0 + r < mi ? U[(int64_t)(ri0 + r0 + r) * lduv + a] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < TS; ++s) {
        const int a = ta + 8 * s;
        if (a < ki) {
          double t = tacc[s];
          for (int r = 0; r < GR; ++r) t = fma(sU[r * LDU + a], sA[r * GQ + tq], t);
          tacc[s] = t;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < TS; ++s) {
      const int a = ta + 8 * s;
      if (a < ki) sT[a * GQ + tq] = tacc[s];
    }
    for (int e = tid; e < GQ * kj; e += GT) {
      const int t = e / kj, c = e - t * kj;
      sV[t * LDU + c] = q0 + t < mj ? V[(int64_t)(cj0 + q0 + t) * lduv + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < CS; ++s) {
      const int e = tid + GT * s;
      if (e < ki * kj) {
        const int a = e / kj, c = e - a * kj;
        double acc = cacc[s];
        for (int t = 0; t < GQ; ++t) acc = fma(sT[a * GQ + t], sV[t * LDU + c], acc);
        cacc[s] = acc;
      }
    }
  }
#pragma unroll
  for (int s = 0; s < CS; ++s) {
    const int e = tid + GT * s;
    if (e < ki * kj) {
      const int a = e / kj, c = e - a * kj;
      core[(int64_t)(roff[i] + a) * ldc + roff[j] + c] = cacc[s];
    }
  }
}

// S_p (KA x m_max, row stride m_max) = sum_{j' in colour(j)} C_ij' V_j'^T,
// columns q < m_j'. CTA per (pair, 64-column tile); thread per (a, q).
__global__ void __launch_bounds__(GT) k_nf_S_gen(const int32_t* __restrict__ off, const int32_t* __restrict__ roff,
                                                 const double* __restrict__ V, int64_t lduv,
                                                 const double* __restrict__ core, int64_t ldc,
                                                 const int32_t* __restrict__ colour, const int32_t* __restrict__ cptr,
                                                 const int32_t* __restrict__ cidx, const int32_t* __restrict__ pair_i,
                                                 const int32_t* __restrict__ nidx, int m_max, int KA,
                                                 double* __restrict__ S) {
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int c = colour[nidx[p]];
  const int ki = roff[i + 1] - roff[i];
  const int q = blockIdx.y * 64 + (threadIdx.x & 63);
  const int a0 = threadIdx.x >> 6;            // rows a0, a0 + 4, ...
  double* Sp = S + (int64_t)p * KA * m_max;
  const double* Crow = core + (int64_t)roff[i] * ldc;
  for (int a = a0; a < ki; a += 4) {
    if (q >= m_max) break;
    double s = 0.0;
    for (int mem = cptr[c]; mem < cptr[c + 1]; ++mem) {
      const int jp = cidx[mem];
      const int kj = roff[jp + 1] - roff[jp];
      if (q >= off[jp + 1] - off[jp]) continue;
      const double* Cij = Crow + (int64_t)a * ldc + roff[jp];
      const double* Vq = V + (int64_t)(off[jp] + q) * lduv;
      for (int e = 0; e < kj; ++e) s = fma(__ldg(&Cij[e]), __ldg(&Vq[e]), s);
    }
    Sp[(int64_t)a * m_max + q] = s;
  }
}

// B_p[r, q] = sum_{j' in colour(j), q < m_j'} A(off_i + r, off_j' + q) - sum_a U_i[r, a] S_p[a, q]
// for q < m_j. CTA per (pair, 32-row tile); threads stride the columns.
template <int KIND>
__global__ void __launch_bounds__(GT) k_nf_B_gen(ublr_op_t op, const int32_t* __restrict__ off,
                                                 const int32_t* __restrict__ roff, int KA,
                                                 const double* __restrict__ U, int64_t lduv,
                                                 const int32_t* __restrict__ colour, const int32_t* __restrict__ cptr,
                                                 const int32_t* __restrict__ cidx, const int32_t* __restrict__ pair_i,
                                                 const int32_t* __restrict__ nidx, const int64_t* __restrict__ b_off,
                                                 int m_max, const double* __restrict__ S, double* __restrict__ B) {
  __shared__ LogTables lt;
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  __syncthreads();
  const int p = blockIdx.x;
  const int i = pair_i[p], j = nidx[p];
  const int c = colour[j];
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int mj = off[j + 1] - off[j];
  const int ki = roff[i + 1] - roff[i];
  const double* Sp = S + (int64_t)p * KA * m_max;
  double* Bp = B + b_off[p];
  for (int rr = 0; rr < 32; ++rr) {
    const int r = blockIdx.y * 32 + rr;
    if (r >= mi) break;
    RowPoint rp = load_row_point(op, ri0 + r, true);
    const double* Ur = U + (int64_t)(ri0 + r) * lduv;
    for (int q = threadIdx.x; q < mj; q += GT) {
      double v = 0.0;
      for (int mem = cptr[c]; mem < cptr[c + 1]; ++mem) {
        const int jp = cidx[mem];
        if (q < off[jp + 1] - off[jp]) v += op_entry<KIND>(op, rp, off[jp] + q, &lt);
      }
      for (int a = 0; a < ki; ++a) v = fma(-__ldg(&Ur[a]), Sp[(int64_t)a * m_max + q], v);
      Bp[(int64_t)r * mj + q] = v;
    }
  }
}

size_t gen_smem(int kmax) {
  return ((size_t)GR * GQ + (size_t)GR * (kmax + 1) + (size_t)kmax * GQ + (size_t)GQ * (kmax + 1)) * sizeof(double) +
         sizeof(LogTables);
}

}  // namespace

// Entry points used by ublr_coupling / ublr_nearfield_colour (coupling.cu)
// when m_max > 256 or k > 64.
int coupling_generic(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k, const double* U,
                     const double* V, int64_t ld_uv, double* core, int64_t ld_c, cudaStream_t st, int m_max, int i0,
                     int i1) {
  const int kk = k < m_max ? k : m_max;
  UBLR_REQUIRE(kk <= GK_MAX, UBLR_ERR_VALUE, "ublr_coupling: rank must be <= 96");
  const size_t smem = gen_smem(kk);
  for (int c0 = i0; c0 < i1; c0 += 65535) {
    const int c1 = c0 + 65535 < i1 ? c0 + 65535 : i1;
    dim3 grid(b, c1 - c0);
    UBLR_DISPATCH_KIND(op->kind, KIND, {
      UBLR_CUDA(cudaFuncSetAttribute(k_coupling_gen<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_coupling_gen<KIND><<<grid, GT, smem, st>>>(*op, off, roff, U, V, ld_uv, core, ld_c, c0, kk);
    });
    UBLR_LAUNCH_CHECK();
  }
  return UBLR_OK;
}

int nearfield_generic(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int k, const double* U,
                      const double* V, int64_t ld_uv, const double* core, int64_t ld_c, const int32_t* colour,
                      const int32_t* cptr, const int32_t* cidx, int m_max, const int32_t* pair_i, const int32_t* nidx,
                      int n_pairs, const int64_t* b_off, double* B, double* S, int KA, cudaStream_t st) {
  UBLR_REQUIRE(n_pairs <= 65535 * 64, UBLR_ERR_VALUE, "ublr_nearfield_colour: too many pairs");
  dim3 gs(n_pairs, (m_max + 63) / 64);
  k_nf_S_gen<<<gs, GT, 0, st>>>(off, roff, V, ld_uv, core, ld_c, colour, cptr, cidx, pair_i, nidx, m_max, KA, S);
  UBLR_LAUNCH_CHECK();
  dim3 gb(n_pairs, (m_max + 31) / 32);
  UBLR_DISPATCH_KIND(op->kind, KIND,
                     (k_nf_B_gen<KIND><<<gb, GT, 0, st>>>(*op, off, roff, KA, U, ld_uv, colour, cptr, cidx, pair_i,
                                                          nidx, b_off, m_max, S, B)));
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

}  // namespace ublr
