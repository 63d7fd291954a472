// K6 / K7 — type-A reconstruction (ref/reconstruction.py:185-244).
//
// K6 `ublr_coupling`: direct_core (ref/reconstruction.py:185-198) pushes the
// K columns of blockdiag(V) through A and projects on U: C = U^T (A V). The
// block-diagonal structure is used directly: C_ij = U_i^T (A_ij V_j), one
// CTA per (i, j), with the A_ij tile generated on the fly (2 m^2 k + 2 m k^2
// flops per pair instead of a dense N x N x K product).
//
// K7 `ublr_nearfield_colour`: structured_identity_discrepancy
// (ref/reconstruction.py:201-244) probes A with one identity per colour, so
// the extracted near block of pair (i, j) is
//   B_ij[:, q] = sum_{j' in colour(j), q < m_j'} (A_ij' - U_i C_ij' V_j'^T)[:, q]
// — the true near residual plus the same-colour far residuals of block row i
// (SURVEY.md F11). Two kernels: S_p = sum_j' C_ij' V_j'^T (k x m, DMMA) per
// pair, then B_p = sum_j' A_ij' - U_i S_p with A generated on the fly.
#include <cstdlib>

#include "common.cuh"
#include "optile.cuh"
#include "gemm_core.cuh"
#include "ws.cuh"

namespace ublr {
namespace {

constexpr int CP_THREADS = 256;
constexpr int CP_BK = 16;

// ---------------------------------------------------------------- coupling
// RW = rows per warp (8 warps cover 8*RW rows >= m_i); NJ = 8-col groups (k <= 8 NJ)
template <int KIND, int RW, int NJ>
__global__ void __launch_bounds__(CP_THREADS) k_coupling(ublr_op_t op, const int32_t* __restrict__ off,
                                                         const int32_t* __restrict__ roff, int k,
                                                         const double* __restrict__ U,
                                                         const double* __restrict__ V, int64_t lduv,
                                                         double* __restrict__ core, int64_t ldc, int i0) {
  constexpr int MR = 8 * RW;          // max rows of block i
  constexpr int SA = MR + 4;          // k-major A tile stride
  constexpr int SB = 8 * NJ + 4;      // V tile stride
  constexpr int RI = RW / 8;          // 8-row groups per warp
  constexpr int SW = 8 * NJ + 1;
  __shared__ LogTables lt;
  extern __shared__ double dsm[];
  double (*As)[CP_BK][SA] = reinterpret_cast<double (*)[CP_BK][SA]>(dsm);
  double (*Bs)[CP_BK][SB] = reinterpret_cast<double (*)[CP_BK][SB]>(dsm + 2 * CP_BK * SA);
  double (*Ws)[SW] = reinterpret_cast<double (*)[SW]>(dsm);  // aliases As/Bs after the k-loop
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);

  const int j = blockIdx.x, i = i0 + blockIdx.y;
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int cj0 = off[j], mj = off[j + 1] - cj0;
  const int ki = roff[i + 1] - roff[i], kj = roff[j + 1] - roff[j];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  // generation: rows r = tid % MR .. (MR <= 256), kk slots
  constexpr int GR = (MR < CP_THREADS) ? MR : CP_THREADS;
  constexpr int GK = CP_THREADS / GR;   // kk lanes
  const int grow = tid % GR;
  const int gk = tid / GR;
  RowPoint rp[(MR + CP_THREADS - 1) / CP_THREADS];
#pragma unroll
  for (int s = 0; s < (MR + CP_THREADS - 1) / CP_THREADS; ++s) {
    int r = grow + s * CP_THREADS;
    rp[s] = load_row_point(op, ri0 + r, r < mi);
  }

  double acc[RI][NJ][2];
#pragma unroll
  for (int a = 0; a < RI; ++a)
#pragma unroll
    for (int b = 0; b < NJ; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  __syncthreads();

  auto stage = [&](int buf, int q0) {
#pragma unroll
    for (int s = 0; s < (MR + CP_THREADS - 1) / CP_THREADS; ++s) {
      for (int kk = gk; kk < CP_BK; kk += GK) {
        int q = q0 + kk;
        double v = 0.0;
        if (rp[s].p >= 0 && q < mj) v = op_entry<KIND>(op, rp[s], cj0 + q, &lt);
        As[buf][kk][grow + s * CP_THREADS] = v;
      }
    }
    for (int e = tid; e < CP_BK * 8 * NJ; e += CP_THREADS) {
      int kk = e / (8 * NJ), c = e - kk * (8 * NJ);
      int q = q0 + kk;
      bool ok = q < mj && c < kj;
      cp_async8(&Bs[buf][kk][c], ok ? (const void*)(V + (int64_t)(cj0 + q) * lduv + c) : (const void*)V, ok);
    }
    cp_async_commit();
  };

  const int nk = (mj + CP_BK - 1) / CP_BK;
  stage(0, 0);
  for (int ks = 0; ks < nk; ++ks) {
    int buf = ks & 1;
    cp_async_wait<0>();
    __syncthreads();
    if (ks + 1 < nk) stage(buf ^ 1, (ks + 1) * CP_BK);
#pragma unroll
    for (int k4 = 0; k4 < CP_BK; k4 += 4) {
      double a[RI], bb[NJ];
#pragma unroll
      for (int s = 0; s < RI; ++s) a[s] = As[buf][k4 + t][warp * RW + s * 8 + g];
#pragma unroll
      for (int c = 0; c < NJ; ++c) bb[c] = Bs[buf][k4 + t][c * 8 + g];
#pragma unroll
      for (int s = 0; s < RI; ++s)
#pragma unroll
        for (int c = 0; c < NJ; ++c) mma8x8x4(acc[s][c][0], acc[s][c][1], a[s], bb[c]);
    }
  }
  // W -> shared (aliases the staging buffers)
  __syncthreads();
#pragma unroll
  for (int s = 0; s < RI; ++s)
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
      int r = warp * RW + s * 8 + g;
      Ws[r][c * 8 + 2 * t] = acc[s][c][0];
      Ws[r][c * 8 + 2 * t + 1] = acc[s][c][1];
    }
  __syncthreads();
  // C_ij = U_i^T W (ki x kj): thread per output, fp64 FMA over the mi rows
  const double* Ui = U + (int64_t)ri0 * lduv;
  for (int e = tid; e < ki * kj; e += CP_THREADS) {
    int a = e / kj, c = e - a * kj;
    double s = 0.0;
    for (int r = 0; r < mi; ++r) s = fma(__ldg(&Ui[(int64_t)r * lduv + a]), Ws[r][c], s);
    core[(int64_t)(roff[i] + a) * ldc + roff[j] + c] = s;
  }
}

// ------------------------------------------------------------- coupling v2
// C_ij = U_i^T (A_ij V_j) per CTA (i, j) on the shared DMMA main loop:
// phase 1 W = A_ij V_j (m_i x k_j, A_ij generated per 32-column k-step,
// V_j rows by cp.async), phase 2 C = U_i^T W with W staged in shared memory
// (k-major) and the 8x8 output tiles of C spread over the warps.
struct OffsetRows {
  int base;
  __device__ __forceinline__ int operator()(int r) const { return base + r; }
};

template <int KIND, class Cfg>
struct CouplingAProducer {
  const ublr_op_t& op;
  const LogTables* lt;
  int cj0, mj;
  RowPoint rp;
  int grow, gk0;
  ColRing<Cfg::BK> ring;
  __device__ CouplingAProducer(const ublr_op_t& op_, const LogTables* lt_, int ri0, int mi, int cj0_, int mj_,
                               double* ringbuf)
      : op(op_), lt(lt_), cj0(cj0_), mj(mj_) {
    grow = threadIdx.x % Cfg::BM;
    gk0 = threadIdx.x / Cfg::BM;
    rp = load_row_point(op, ri0 + grow, grow < mi);
    ring.buf = ringbuf;
  }
  __device__ __forceinline__ void prefetch(int ks) {
    if (KIND != UBLR_OP_DENSE) ring.prefetch(op, ks, cj0 + ks * Cfg::BK, cj0 + mj, Cfg::NT);
  }
  __device__ __forceinline__ void stage(double* As, int ks) { stage_part(As, ks, 0, 1); }
  __device__ __forceinline__ void stage_part(double* As, int ks, int part, int nparts) {
    constexpr int KL = Cfg::NT / Cfg::BM;
    constexpr int E = Cfg::BK / KL;
    int e0, e1;
    chunk_range<E, 2>(part, nparts, e0, e1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e < e0 || e >= e1) continue;
      int kk = gk0 + e * KL;
      int q = ks * Cfg::BK + kk;
      double v = 0.0;
      if (rp.p >= 0 && q < mj) {
        if (KIND == UBLR_OP_DENSE) v = op_entry<KIND>(op, rp, cj0 + q, lt);
        else v = kernel_entry<KIND>(op, rp, cj0 + q, ring.at(ks, 0, kk), ring.at(ks, 1, kk), ring.at(ks, 2, kk), lt);
      }
      As[Cfg::ai(grow, kk)] = v;
    }
  }
};

template <class Cfg>
struct CouplingBProducer {
  const double* V;
  int64_t ld;
  int cj0, mj, kj;
  bool vec2;
  __device__ __forceinline__ void stage(double* Bs, int ks) {
    tile_copy<Cfg::NT>(Bs, Cfg::SB, V, ld, Cfg::BK, Cfg::BN, ks * Cfg::BK, 0, mj, kj, OffsetRows{cj0}, vec2);
  }
};

template <int KIND, class Cfg>
__global__ void __launch_bounds__(Cfg::NT) k_coupling2(ublr_op_t op, const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ roff, const double* __restrict__ U,
                                                       const double* __restrict__ V, int64_t lduv,
                                                       double* __restrict__ core, int64_t ldc, int i0, int vec2) {
  static_assert(Cfg::WNW == 1, "each warp owns whole rows of W");
  constexpr int BN = Cfg::BN;
  constexpr int NJ2 = BN / 8;
  constexpr int SW = BN + 4;
  __shared__ LogTables lt;
  __shared__ double ringbuf[9 * Cfg::BK];
  extern __shared__ double dsm[];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int j = blockIdx.x, i = i0 + blockIdx.y;
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int cj0 = off[j], mj = off[j + 1] - cj0;
  const int ki = roff[i + 1] - roff[i], kj = roff[j + 1] - roff[j];
  CouplingAProducer<KIND, Cfg> ap(op, &lt, ri0, mi, cj0, mj, ringbuf);
  CouplingBProducer<Cfg> bp{V, lduv, cj0, mj, kj, vec2 != 0};
  double acc[Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a)
#pragma unroll
    for (int c = 0; c < Cfg::NJ; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  __syncthreads();
  dmma_mainloop<Cfg>(ap, bp, (mj + Cfg::BK - 1) / Cfg::BK, dsm, acc);
  __syncthreads();
  // W -> shared, k-major (row r of W = k index of C = U^T W)
  double* Ws = dsm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a)
#pragma unroll
    for (int c = 0; c < Cfg::NJ; ++c) {
      int r = warp * Cfg::WM + a * 8 + g;
      Ws[r * SW + c * 8 + 2 * t] = acc[a][c][0];
      Ws[r * SW + c * 8 + 2 * t + 1] = acc[a][c][1];
    }
  __syncthreads();
  // C = U_i^T W : (ki x kj) in 8x8 tiles, tile ids spread over the warps
  constexpr int NW = Cfg::NT / 32;
  const int mt = (ki + 7) / 8, nt = (kj + 7) / 8;
  // U_i -> shared (behind W), so phase 2 reads both operands from shared memory
  constexpr int SU = BN + 1;
  double* Us = dsm + Cfg::BM * SW;
  const double* Ui = U + (int64_t)ri0 * lduv;
  for (int e = threadIdx.x; e < mi * ki; e += Cfg::NT) {
    int r = e / ki, a = e - r * ki;
    Us[r * SU + a] = Ui[(int64_t)r * lduv + a];
  }
  __syncthreads();
  constexpr int MAXT = (8 * NJ2 + NW - 1) / NW;  // tiles per warp when ki, kj <= BN
  double c2[MAXT][2];
#pragma unroll
  for (int q = 0; q < MAXT; ++q) c2[q][0] = c2[q][1] = 0.0;
  for (int r0 = 0; r0 < mi; r0 += 4) {
    const int r = r0 + t;
    const bool rok = r < mi;
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
      int tile = warp + q * NW;
      if (tile >= mt * nt) break;
      int ta = tile / nt, tc = tile - (tile / nt) * nt;
      int acol = ta * 8 + g;
      double av = (rok && acol < ki) ? Us[r * SU + acol] : 0.0;
      double bv = rok ? Ws[r * SW + tc * 8 + g] : 0.0;
      mma8x8x4(c2[q][0], c2[q][1], av, bv);
    }
  }
#pragma unroll
  for (int q = 0; q < MAXT; ++q) {
    int tile = warp + q * NW;
    if (tile >= mt * nt) break;
    int ta = tile / nt, tc = tile - (tile / nt) * nt;
    int a = ta * 8 + g;
    int c = tc * 8 + 2 * t;
    if (a < ki) {
      double* dst = core + (int64_t)(roff[i] + a) * ldc + roff[j];
      if (c < kj) dst[c] = c2[q][0];
      if (c + 1 < kj) dst[c + 1] = c2[q][1];
    }
  }
}

// ------------------------------------------------------------- coupling v3
// Warp-specialised coupling for kernel operators with m <= 256, k <= 48
// (configs 3-5). One CTA per (row block i, chunk of column blocks j):
//   phase 1  T = U_i^T A_ij  (KP x 256): producer warps cp.async the k-slices
//            of U_i and generate A_ij eight block-i rows at a time into a
//            5-stage mbarrier ring; consumer warps (2 x 4, 24 x 64 tiles) run
//            the DMMAs;
//   phase 2  C_ij = T V_j   (KP x k_j): the A fragments come straight from the
//            phase-1 accumulators by quad shuffles, V_j is staged in shared
//            memory by the producers during phase 1; the four column-warp
//            partials are summed in a fixed order (shared memory, aliasing
//            V_j) and written to the core.
// The producers run ahead into the next j while the consumers do phase 2.
// Entries are generated as A(i_r, j_q) = k(x_jq - x_ir): the squared distance
// is bitwise that of the row-major apply (negated differences).
struct Cp3 {
  static constexpr int BK = 8, STAGES = 5, KP = 48, NQ = 256;
  static constexpr int NPROD = 256, NCONS = 256, NT = NPROD + NCONS;
  static constexpr int SA = KP + 4, SB = NQ + 4, SV = KP + 4;
  static constexpr int A_STAGE = BK * SA, B_STAGE = BK * SB;
  static constexpr int WMW = 2, WNW = 4, WM = KP / WMW, WN = NQ / WNW, MI = WM / 8, NJ = WN / 8, NC = KP / 8;
  static constexpr int CONS_REGS = 200, PROD_REGS = 56;
  static constexpr size_t smem_bytes() {
    return (size_t)(STAGES * (A_STAGE + B_STAGE) + NQ * SV + 3 * NQ) * sizeof(double);
  }
  static_assert(4 * KP * KP <= NQ * SV, "phase-2 partials alias the V_j buffer");
};

template <int KIND, int DIM>
__global__ void __launch_bounds__(Cp3::NT, 1) k_coupling3(ublr_op_t op, const int32_t* __restrict__ off,
                                                          const int32_t* __restrict__ roff,
                                                          const double* __restrict__ U,
                                                          const double* __restrict__ V, int64_t lduv,
                                                          double* __restrict__ core, int64_t ldc, int i0, int b,
                                                          int jchunk, int vec2) {
  using C = Cp3;
  constexpr int BK = C::BK, STAGES = C::STAGES, KP = C::KP, NQ = C::NQ, SA = C::SA, SB = C::SB, SV = C::SV;
  constexpr int MI = C::MI, NJ = C::NJ, NC = C::NC;
  __shared__ LogTables lt;
  __shared__ uint64_t full[STAGES], empty[STAGES], vfull, vempty;
  extern __shared__ double dsm[];
  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * C::A_STAGE;
  double* Vs = Bs0 + STAGES * C::B_STAGE;
  double* xi = Vs + NQ * SV;  // coordinates of block i's points, [3][NQ]
  const int i = i0 + blockIdx.x;
  const int j0 = blockIdx.y * jchunk;
  const int j1 = min(b, j0 + jchunk);
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int ki = roff[i + 1] - roff[i];
  const int nk = (mi + BK - 1) / BK;
  const int n = (int)op.n;
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  for (int e = threadIdx.x; e < 3 * NQ; e += C::NT) {
    const int a = e / NQ, r = e - a * NQ;
    xi[e] = (r < mi && a < DIM) ? op.coords[(int64_t)a * n + ri0 + r] : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ws::mbar_init(&full[s], 2 * C::NPROD);  // cp.async (U slice) + generator arrivals
      ws::mbar_init(&empty[s], C::NCONS);
    }
    ws::mbar_init(&vfull, C::NPROD);
    ws::mbar_init(&vempty, C::NCONS);
  }
  __syncthreads();

  if (threadIdx.x < C::NPROD) {
    // ---------------- producers: one column q of block j each
    ws::regs_dec<C::PROD_REGS>();
    const int q = threadIdx.x;
    const double diag = op.diag;
    int it = 0;
    for (int j = j0; j < j1; ++j) {
      const int jl = j - j0;
      const int cj0 = off[j], mj = off[j + 1] - cj0, kj = roff[j + 1] - roff[j];
      const bool qok = q < mj;
      const RowPoint rp = load_row_point(op, qok ? cj0 + q : cj0, true);
      for (int ks = 0; ks < nk; ++ks, ++it) {
        const int s = it % STAGES;
        ws::mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1) ^ 1);
        tile_copy<C::NPROD>(As0 + s * C::A_STAGE, SA, U, lduv, BK, KP, ks * BK, 0, mi, ki, OffsetRows{ri0},
                            vec2 != 0);
        cp_async_commit();
        ws::mbar_cp_async_arrive(&full[s]);
        double v[BK];
#pragma unroll
        for (int e = 0; e < BK; ++e) {
          const int r = ks * BK + e;
          const double a = kernel_entry_dim<KIND, DIM>(rp, ri0 + r, xi[r], DIM > 1 ? xi[NQ + r] : 0.0,
                                                       DIM > 2 ? xi[2 * NQ + r] : 0.0, diag, &lt);
          v[e] = (qok && r < mi) ? a : 0.0;
        }
        double* Bs = Bs0 + s * C::B_STAGE;
#pragma unroll
        for (int e = 0; e < BK; ++e) Bs[e * SB + q] = v[e];
        ws::mbar_arrive(&full[s]);
        if (ks == min(2, nk - 1)) {
          // V_j for phase 2, once the consumers have released phase 2 of j - 1
          ws::mbar_wait(&vempty, ((uint32_t)jl & 1) ^ 1);
          tile_copy<C::NPROD>(Vs, SV, V, lduv, NQ, KP, 0, 0, mj, kj, OffsetRows{cj0}, vec2 != 0);
          cp_async_commit();
          ws::mbar_cp_async_arrive(&vfull);
        }
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers
  ws::regs_inc<C::CONS_REGS>();
  const int ct = threadIdx.x - C::NPROD;
  const int warp = ct >> 5, lane = ct & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / C::WNW, wc = warp % C::WNW;
  const int am0 = wr * C::WM + g, bn0 = wc * C::WN + g;
  double acc[MI][NJ][2];
#pragma unroll
  for (int a = 0; a < MI; ++a)
#pragma unroll
    for (int c = 0; c < NJ; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  int it = 0;
  for (int j = j0; j < j1; ++j) {
    const int jl = j - j0;
    for (int ks = 0; ks < nk; ++ks, ++it) {
      const int s = it % STAGES;
      ws::mbar_wait(&full[s], (uint32_t)(it / STAGES) & 1);
      const double* As = As0 + s * C::A_STAGE;
      const double* Bs = Bs0 + s * C::B_STAGE;
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        const int kr = k4 * 4 + t;
        double av[MI], bv[NJ];
#pragma unroll
        for (int a = 0; a < MI; ++a) av[a] = As[kr * SA + am0 + a * 8];
#pragma unroll
        for (int c = 0; c < NJ; ++c) bv[c] = Bs[kr * SB + bn0 + c * 8];
#pragma unroll
        for (int a = 0; a < MI; ++a)
#pragma unroll
          for (int c = 0; c < NJ; ++c) mma8x8x4(acc[a][c][0], acc[a][c][1], av[a], bv[c]);
      }
      ws::mbar_arrive(&empty[s]);
    }
    // phase 2: partial C (rows of this warp) over this warp's 64 columns q
    ws::mbar_wait(&vfull, (uint32_t)jl & 1);
    double cp[MI][NC][2];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int c = 0; c < NC; ++c) cp[a][c][0] = cp[a][c][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int src = (g << 2) + 2 * h + (t >> 1);
        double av[MI];
#pragma unroll
        for (int a = 0; a < MI; ++a) {
          const double v0 = __shfl_sync(0xffffffffu, acc[a][c][0], src);
          const double v1 = __shfl_sync(0xffffffffu, acc[a][c][1], src);
          av[a] = (t & 1) ? v1 : v0;
        }
        const double* vrow = Vs + (wc * C::WN + c * 8 + 4 * h + t) * SV + g;
#pragma unroll
        for (int nn = 0; nn < NC; ++nn) {
          const double bvv = vrow[nn * 8];
#pragma unroll
          for (int a = 0; a < MI; ++a) mma8x8x4(cp[a][nn][0], cp[a][nn][1], av[a], bvv);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int c = 0; c < NJ; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    ws::named_sync(2, C::NCONS);  // every consumer is done reading V_j
    double* red = Vs;             // [wc][KP][KP]
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int nn = 0; nn < NC; ++nn) {
        const int ra = wr * C::WM + a * 8 + g, cc = nn * 8 + 2 * t;
        red[(wc * KP + ra) * KP + cc] = cp[a][nn][0];
        red[(wc * KP + ra) * KP + cc + 1] = cp[a][nn][1];
      }
    ws::named_sync(2, C::NCONS);
    const int kj = roff[j + 1] - roff[j];
    double* crow = core + (int64_t)roff[i] * ldc + roff[j];
    for (int e = ct; e < ki * kj; e += C::NCONS) {
      const int a = e / kj, c = e - a * kj;
      const int o = a * KP + c;
      const double sum = ((red[o] + red[KP * KP + o]) + red[2 * KP * KP + o]) + red[3 * KP * KP + o];
      crow[(int64_t)a * ldc + c] = sum;
    }
    ws::mbar_arrive(&vempty);
  }
}

// ------------------------------------------------------- near field: S_p
// S_p (k x m_max) = sum_{j' in colour(j)} C_{i j'} V_{j'}^T, columns q < m_j'.
// One CTA per near pair; 8 warps split the m_max columns, each warp holds
// all k rows x (m_max / 8) columns of accumulators.
template <int NA, int NQ>
__global__ void __launch_bounds__(CP_THREADS) k_nf_S(const int32_t* __restrict__ off,
                                                     const int32_t* __restrict__ roff,
                                                     const double* __restrict__ V, int64_t lduv,
                                                     const double* __restrict__ core, int64_t ldc,
                                                     const int32_t* __restrict__ colour,
                                                     const int32_t* __restrict__ cptr,
                                                     const int32_t* __restrict__ cidx,
                                                     const int32_t* __restrict__ pair_i,
                                                     const int32_t* __restrict__ nidx, int m_max,
                                                     double* __restrict__ S) {
  // NA: 8-row groups of k (k <= 8 NA); NQ: 8-col groups per warp (m_max <= 64 NQ)
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int c = colour[nidx[p]];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ki = roff[i + 1] - roff[i];
  double acc[NA][NQ][2];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[a][q][0] = acc[a][q][1] = 0.0;
  const double* Crow = core + (int64_t)roff[i] * ldc;
  for (int mem = cptr[c]; mem < cptr[c + 1]; ++mem) {
    const int jp = cidx[mem];
    const int kj = roff[jp + 1] - roff[jp];
    const int mj = off[jp + 1] - off[jp];
    const double* Vj = V + (int64_t)off[jp] * lduv;
    const double* Cij = Crow + roff[jp];
    for (int e0 = 0; e0 < kj; e0 += 4) {
      int e = e0 + t;
      double a[NA], bb[NQ];
#pragma unroll
      for (int s = 0; s < NA; ++s) {
        int row = s * 8 + g;
        a[s] = (row < ki && e < kj) ? __ldg(&Cij[(int64_t)row * ldc + e]) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        int col = (warp * NQ + q) * 8 + g;
        bb[q] = (col < mj && e < kj) ? __ldg(&Vj[(int64_t)col * lduv + e]) : 0.0;
      }
#pragma unroll
      for (int s = 0; s < NA; ++s)
#pragma unroll
        for (int q = 0; q < NQ; ++q) mma8x8x4(acc[s][q][0], acc[s][q][1], a[s], bb[q]);
    }
  }
  double* Sp = S + (int64_t)p * (8 * NA) * m_max;
#pragma unroll
  for (int s = 0; s < NA; ++s)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      int row = s * 8 + g;
      int col = (warp * NQ + q) * 8 + 2 * t;
      if (col < m_max) Sp[(int64_t)row * m_max + col] = acc[s][q][0];
      if (col + 1 < m_max) Sp[(int64_t)row * m_max + col + 1] = acc[s][q][1];
    }
}

// ------------------------------------------------------- near field: B_p
// CTA per (pair p, tile of 32 rows): thread owns column q = tid % QW and
// rows tid / QW + s * (256 / QW).
template <int KIND>
__global__ void __launch_bounds__(CP_THREADS) k_nf_B(ublr_op_t op, const int32_t* __restrict__ off,
                                                     const int32_t* __restrict__ roff, int KA,
                                                     const double* __restrict__ U, int64_t lduv,
                                                     const int32_t* __restrict__ colour,
                                                     const int32_t* __restrict__ cptr,
                                                     const int32_t* __restrict__ cidx,
                                                     const int32_t* __restrict__ pair_i,
                                                     const int32_t* __restrict__ nidx,
                                                     const int64_t* __restrict__ b_off, int m_max,
                                                     const double* __restrict__ S, double* __restrict__ B) {
  constexpr int RT = 32;
  __shared__ LogTables lt;
  __shared__ double rowc[3][RT];
  __shared__ int rowo[RT];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int jn = nidx[p];
  const int c = colour[jn];
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int mjn = off[jn + 1] - off[jn];
  const int r0 = blockIdx.y * RT;
  if (r0 >= mi) return;
  const int ki = roff[i + 1] - roff[i];
  const int tid = threadIdx.x;
  const int QW = m_max < CP_THREADS ? m_max : CP_THREADS;  // m_max <= 256 enforced by host
  const int q = tid % QW;
  const int rstep = CP_THREADS / QW;
  const int r_first = tid / QW;
  const bool active = tid < rstep * QW;
  if (tid < RT) {
    int p_row = ri0 + r0 + tid;
    bool ok = r0 + tid < mi;
    if (KIND == UBLR_OP_DENSE) {
      rowo[tid] = ok ? (op.perm ? op.perm[p_row] : p_row) : 0;
    } else {
      rowo[tid] = ok ? p_row : -1;
      for (int a = 0; a < 3; ++a) rowc[a][tid] = (ok && a < op.dim) ? op.coords[(int64_t)a * op.n + p_row] : 0.0;
    }
  }
  __syncthreads();
  if (!active) return;
  constexpr int MAXS = RT;  // rows per thread upper bound (QW >= 8 assumed)
  double asum[MAXS];
  const int nrows = (RT + rstep - 1) / rstep;
#pragma unroll
  for (int s = 0; s < MAXS; ++s) asum[s] = 0.0;
  for (int mem = cptr[c]; mem < cptr[c + 1]; ++mem) {
    const int jp = cidx[mem];
    const int mj = off[jp + 1] - off[jp];
    if (q >= mj) continue;
    const int col = off[jp] + q;
    // column point
    RowPoint cp = load_row_point(op, col, true);
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      if (s >= nrows) break;
      int r = r_first + s * rstep;
      if (r >= RT || r0 + r >= mi) continue;
      double v;
      if (KIND == UBLR_OP_DENSE) {
        v = op.transpose ? op.A[(int64_t)cp.orig * op.lda + rowo[r]] : op.A[(int64_t)rowo[r] * op.lda + cp.orig];
      } else {
        if (rowo[r] == col) {
          v = op.diag;
        } else {
          double d = rowc[0][r] - cp.x0;
          double r2 = d * d;
          if (op.dim > 1) { d = rowc[1][r] - cp.x1; r2 = fma(d, d, r2); }
          if (op.dim > 2) { d = rowc[2][r] - cp.x2; r2 = fma(d, d, r2); }
          v = (KIND == UBLR_OP_LOG) ? -0.5 * fast_log(r2, &lt) : rsqrt(r2);
        }
      }
      asum[s] += v;
    }
  }
  if (q >= mjn) return;
  const double* Sp = S + (int64_t)p * KA * m_max;
  double* Bp = B + b_off[p];
  for (int s = 0; s < nrows; ++s) {
    int r = r_first + s * rstep;
    if (r >= RT || r0 + r >= mi) continue;
    const double* urow = U + (int64_t)(ri0 + r0 + r) * lduv;
    double v = asum[s];
    for (int a = 0; a < ki; ++a) v = fma(-__ldg(&urow[a]), Sp[(int64_t)a * m_max + q], v);
    Bp[(int64_t)(r0 + r) * mjn + q] = v;
  }
}


// ------------------------------------------------- near field v3 (m <= 256)
// S_p = sum_{j' in colour} C_ij' V_j'^T as one GEMM per pair: K runs over
// (member j', b) in BK = 16 slices, A = the C_ij' slices (rows of the core,
// m-major cp.async), B = V_j'^T (n-major: V_j' rows), on the shared DMMA
// main loop. 48 x 256 CTA tile, 8 warps of 24 x 64.
constexpr int NFS_KP = 48;
using NfsCfg = TileCfg<NFS_KP, 256, 16, 2, 4, 3, false, false>;

struct NfSA {
  const double* crow; int64_t ldc; const int32_t* cidx; const int32_t* roff; int mem0, ki; bool vec;
  __device__ __forceinline__ void stage(double* As, int ks) {
    constexpr int KS = NFS_KP / NfsCfg::BK;
    const int jp = cidx[mem0 + ks / KS], b0 = (ks % KS) * NfsCfg::BK;
    const int kj = roff[jp + 1] - roff[jp];
    tile_copy<NfsCfg::NT>(As, NfsCfg::SA, crow + roff[jp] + b0, ldc, NfsCfg::BM, NfsCfg::BK, 0, 0, ki, kj - b0,
                          IdentityRows{}, vec);
  }
};
struct NfSB {
  const double* V; int64_t lduv; const int32_t* cidx; const int32_t* off; const int32_t* roff; int mem0; bool vec;
  __device__ __forceinline__ void stage(double* Bs, int ks) {
    constexpr int KS = NFS_KP / NfsCfg::BK;
    const int jp = cidx[mem0 + ks / KS], b0 = (ks % KS) * NfsCfg::BK;
    const int kj = roff[jp + 1] - roff[jp], mj = off[jp + 1] - off[jp];
    tile_copy<NfsCfg::NT>(Bs, NfsCfg::SB, V + (int64_t)off[jp] * lduv + b0, lduv, NfsCfg::BN, NfsCfg::BK, 0, 0, mj,
                          kj - b0, IdentityRows{}, vec);
  }
};

__global__ void __launch_bounds__(NfsCfg::NT) k_nf_S3(const int32_t* __restrict__ off,
                                                      const int32_t* __restrict__ roff,
                                                      const double* __restrict__ V, int64_t lduv,
                                                      const double* __restrict__ core, int64_t ldc,
                                                      const int32_t* __restrict__ colour,
                                                      const int32_t* __restrict__ cptr,
                                                      const int32_t* __restrict__ cidx,
                                                      const int32_t* __restrict__ pair_i,
                                                      const int32_t* __restrict__ nidx, int m_max, int KA,
                                                      double* __restrict__ S, int vec) {
  using Cfg = NfsCfg;
  extern __shared__ double dsm[];
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int c = colour[nidx[p]];
  const int ki = roff[i + 1] - roff[i];
  const int mem0 = cptr[c], nmem = cptr[c + 1] - mem0;
  NfSA ap{core + (int64_t)roff[i] * ldc, ldc, cidx, roff, mem0, ki, vec != 0};
  NfSB bp{V, lduv, cidx, off, roff, mem0, vec != 0};
  double acc[Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::NJ; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  WholeStage<NfSA> apw{ap};
  dmma_mainloop<Cfg>(apw, bp, nmem * (NFS_KP / Cfg::BK), dsm, acc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
  double* Sp = S + (int64_t)p * KA * m_max;
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a) {
    const int row = wr * Cfg::WM + a * 8 + g;
    if (row >= KA) continue;
#pragma unroll
    for (int b = 0; b < Cfg::NJ; ++b) {
      const int q = wc * Cfg::WN + b * 8 + 2 * t;
      if (q < m_max) Sp[(int64_t)row * m_max + q] = acc[a][b][0];
      if (q + 1 < m_max) Sp[(int64_t)row * m_max + q + 1] = acc[a][b][1];
    }
  }
}

// B_p[r][q] = sum_{j' in colour} A(i_r, j'_q) - (U_i S_p)[r][q]: thread = column
// q, 16 rows per CTA; the next member's column point is loaded one member
// ahead, the row points of the slab are shared-memory broadcasts, and the
// diagonal select is only evaluated for the member j' = i.
constexpr int NFB_RT = 16;  // rows per CTA (accumulators + broadcast row points stay in registers)
template <int KIND, int DIM>
__global__ void __launch_bounds__(256, 2) k_nf_B3(ublr_op_t op, const int32_t* __restrict__ off,
                                               const int32_t* __restrict__ roff, int KA,
                                               const double* __restrict__ U, int64_t lduv,
                                               const int32_t* __restrict__ colour,
                                               const int32_t* __restrict__ cptr,
                                               const int32_t* __restrict__ cidx,
                                               const int32_t* __restrict__ pair_i,
                                               const int32_t* __restrict__ nidx,
                                               const int64_t* __restrict__ b_off, int m_max,
                                               const double* __restrict__ S, double* __restrict__ B) {
  constexpr int RT = NFB_RT;
  __shared__ LogTables lt;
  __shared__ double xr[DIM][RT];
  __shared__ double us[RT][65];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int p = blockIdx.x;
  const int i = pair_i[p];
  const int jn = nidx[p];
  const int c = colour[jn];
  const int ri0 = off[i], mi = off[i + 1] - ri0;
  const int mjn = off[jn + 1] - off[jn];
  const int r0 = blockIdx.y * RT;
  if (r0 >= mi) return;
  const int ki = roff[i + 1] - roff[i];
  const int q = threadIdx.x;
  const int n = (int)op.n;
  for (int e = threadIdx.x; e < DIM * RT; e += blockDim.x) {
    const int a = e / RT, r = e - a * RT;
    xr[a][r] = (r0 + r < mi) ? op.coords[(int64_t)a * n + ri0 + r0 + r] : 0.0;
  }
  for (int e = threadIdx.x; e < RT * ki; e += blockDim.x) {
    const int r = e / ki, a = e - r * ki;
    us[r][a] = (r0 + r < mi) ? U[(int64_t)(ri0 + r0 + r) * lduv + a] : 0.0;
  }
  __syncthreads();
  double acc[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) acc[r] = 0.0;
  const int mem0 = cptr[c], mem1 = cptr[c + 1];
  const double diag = op.diag;
  // column point of member mem (one ahead)
  auto colpt = [&](int mem, double (&x)[DIM], int& col, bool& ok) {
    const int jp = cidx[mem];
    ok = q < off[jp + 1] - off[jp];
    col = off[jp] + (ok ? q : 0);
#pragma unroll
    for (int a = 0; a < DIM; ++a) x[a] = op.coords[(int64_t)a * n + col];
  };
  double xc[DIM], xn[DIM];
  int colc, coln = 0;
  bool okc, okn = false;
  colpt(mem0, xc, colc, okc);
  for (int mem = mem0; mem < mem1; ++mem) {
    if (mem + 1 < mem1) colpt(mem + 1, xn, coln, okn);
    if (okc) {
      const bool self = cidx[mem] == i;
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        double d = xr[0][r] - xc[0];
        double r2 = d * d;
        if (DIM > 1) {
          d = xr[1][r] - xc[1];
          r2 = fma(d, d, r2);
        }
        if (DIM > 2) {
          d = xr[2][r] - xc[2];
          r2 = fma(d, d, r2);
        }
        double v = (KIND == UBLR_OP_LOG) ? -0.5 * fast_log(r2, &lt) : rsqrt(r2);
        if (self && ri0 + r0 + r == colc) v = diag;
        acc[r] += v;
      }
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) xc[a] = xn[a];
    colc = coln;
    okc = okn;
  }
  if (q >= mjn) return;
  const double* Sp = S + (int64_t)p * KA * m_max;
  double* Bp = B + b_off[p];
  for (int a = 0; a < ki; ++a) {
    const double sa = Sp[(int64_t)a * m_max + q];
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r] = fma(-us[r][a], sa, acc[r]);
  }
#pragma unroll
  for (int r = 0; r < RT; ++r)
    if (r0 + r < mi) Bp[(int64_t)(r0 + r) * mjn + q] = acc[r];
}
}  // namespace
}  // namespace ublr

using namespace ublr;

namespace ublr {
int coupling_generic(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k, const double* U,
                     const double* V, int64_t ld_uv, double* core, int64_t ld_c, cudaStream_t st, int m_max, int i0,
                     int i1);
int nearfield_generic(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int k, const double* U,
                      const double* V, int64_t ld_uv, const double* core, int64_t ld_c, const int32_t* colour,
                      const int32_t* cptr, const int32_t* cidx, int m_max, const int32_t* pair_i, const int32_t* nidx,
                      int n_pairs, const int64_t* b_off, double* B, double* S, int KA, cudaStream_t st);
}  // namespace ublr

static size_t coupling_smem(int MR, int NJ) {
  size_t stage = (size_t)2 * CP_BK * (MR + 4) + (size_t)2 * CP_BK * (8 * NJ + 4);
  size_t w = (size_t)MR * (8 * NJ + 1);
  return (stage > w ? stage : w) * sizeof(double);
}

extern "C" int ublr_coupling(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                             const double* U, const double* V, int64_t ld_uv, double* core, int64_t ld_c,
                             void* stream, int m_max, int i0, int i1) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && roff && U && V && core && k >= 1 && ld_uv >= k, UBLR_ERR_VALUE,
               "ublr_coupling: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  UBLR_REQUIRE(0 <= i0 && i0 < i1 && i1 <= b, UBLR_ERR_VALUE, "ublr_coupling: bad block-row range");
  int kk = k < m_max ? k : m_max;  // effective ranks never exceed min(k, m)
  // blocks above 256 points or ranks above 64: the general kernel (coupling_gen.cu)
  if (m_max > 256 || kk > 64) return coupling_generic(op, off, roff, b, k, U, V, ld_uv, core, ld_c, st, m_max, i0, i1);
  UBLR_REQUIRE(b <= 65535, UBLR_ERR_VALUE, "ublr_coupling: b <= 65535");
  int vec2 = ((ld_uv % 2) == 0 && ((uintptr_t)V) % 16 == 0) ? 1 : 0;
  static const int cp_ver = [] {
    const char* e = getenv("UBLR_COUPLING_VERSION");
    return e ? atoi(e) : 3;
  }();
  if (cp_ver == 3 && op->kind != UBLR_OP_DENSE && m_max > 64 && m_max <= Cp3::NQ && kk <= Cp3::KP) {
    // column-block chunks per CTA: enough CTAs for the 148 SMs, long runs per CTA
    const int rows = i1 - i0;
    int chunks = (148 * 4 + rows - 1) / rows;
    if (chunks > b) chunks = b;
    const int jchunk = (b + chunks - 1) / chunks;
    dim3 g3((unsigned)rows, (unsigned)((b + jchunk - 1) / jchunk));
    const int v2 = vec2 && ((uintptr_t)U) % 16 == 0;
    size_t sm = Cp3::smem_bytes();
#define UBLR_CP3(KIND, DIM)                                                                                     \
  {                                                                                                             \
    UBLR_CUDA(cudaFuncSetAttribute(k_coupling3<KIND, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_coupling3<KIND, DIM><<<g3, Cp3::NT, sm, st>>>(*op, off, roff, U, V, ld_uv, core, ld_c, i0, b, jchunk, v2);  \
  }
    if (op->kind == UBLR_OP_LOG) {
      if (op->dim == 1) UBLR_CP3(UBLR_OP_LOG, 1) else if (op->dim == 2) UBLR_CP3(UBLR_OP_LOG, 2) else UBLR_CP3(UBLR_OP_LOG, 3)
    } else {
      if (op->dim == 1) UBLR_CP3(UBLR_OP_INV, 1) else if (op->dim == 2) UBLR_CP3(UBLR_OP_INV, 2) else UBLR_CP3(UBLR_OP_INV, 3)
    }
#undef UBLR_CP3
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
  dim3 grid(b, i1 - i0);
#define UBLR_CP2(BM, BN)                                                                                     \
  UBLR_DISPATCH_KIND(op->kind, KIND, {                                                                      \
    using Cfg = TileCfg<BM, BN, 32, 8, 1, 2>;                                                               \
    size_t sm = Cfg::smem_bytes();                                                                          \
    size_t sw = (size_t)(BM) * ((BN) + 4 + (BN) + 1) * sizeof(double);  /* W and U_i after the main loop */  \
    if (sw > sm) sm = sw;                                                                                   \
    UBLR_CUDA(cudaFuncSetAttribute(k_coupling2<KIND, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_coupling2<KIND, Cfg><<<grid, Cfg::NT, sm, st>>>(*op, off, roff, U, V, ld_uv, core, ld_c, i0, vec2);     \
  })
  if (m_max <= 64) {
    if (kk <= 16) { UBLR_CP2(64, 16); }
    else if (kk <= 24) { UBLR_CP2(64, 24); }
    else if (kk <= 48) { UBLR_CP2(64, 48); }
    else { UBLR_CP2(64, 64); }
  } else {
    if (kk <= 16) { UBLR_CP2(256, 16); }
    else if (kk <= 24) { UBLR_CP2(256, 24); }
    else if (kk <= 48) { UBLR_CP2(256, 48); }
    else { UBLR_CP2(256, 64); }
  }
#undef UBLR_CP2
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

static int ka_of(int k) { return (k <= 8) ? 8 : (k <= 16) ? 16 : (k <= 32) ? 32 : (k <= 64) ? 64 : (k + 7) / 8 * 8; }

extern "C" int64_t ublr_nearfield_workspace_bytes(int n_pairs, int k, int m_max) {
  return (int64_t)n_pairs * ka_of(k) * m_max * (int64_t)sizeof(double);
}

extern "C" int ublr_nearfield_colour(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                                     const double* U, const double* V, int64_t ld_uv, const double* core,
                                     int64_t ld_c, const int32_t* colour, const int32_t* cptr, const int32_t* cidx,
                                     int n_colours, int m_max, const int32_t* pair_i, const int32_t* nidx,
                                     int n_pairs, const int64_t* b_off, double* B, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && n_colours > 0 && n_pairs > 0 && off && roff && U && V && core && colour && cptr && cidx &&
                   pair_i && nidx && b_off && B && workspace,
               UBLR_ERR_VALUE, "ublr_nearfield_colour: bad arguments");
  UBLR_REQUIRE(workspace_bytes >= ublr_nearfield_workspace_bytes(n_pairs, k, m_max), UBLR_ERR_VALUE,
               "ublr_nearfield_colour: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double* S = (double*)workspace;
  const int KA = ka_of(k);
  if (m_max > 256 || k > 64)   // the general kernels (coupling_gen.cu)
    return nearfield_generic(op, off, roff, k, U, V, ld_uv, core, ld_c, colour, cptr, cidx, m_max, pair_i, nidx, n_pairs,
                             b_off, B, S, KA, st);
  static const int nf_ver = [] {
    const char* e = getenv("UBLR_NEARFIELD_VERSION");
    return e ? atoi(e) : 3;
  }();
  const int kk = k < m_max ? k : m_max;
  if (nf_ver == 3 && op->kind != UBLR_OP_DENSE && m_max > 64 && kk <= NFS_KP) {
    const int vec = ((ld_uv % 2) == 0 && (ld_c % 2) == 0 && (k % 2) == 0 && ((uintptr_t)V) % 16 == 0 &&
                     ((uintptr_t)core) % 16 == 0) ? 1 : 0;
    size_t sm = NfsCfg::smem_bytes();
    UBLR_CUDA(cudaFuncSetAttribute(k_nf_S3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_nf_S3<<<n_pairs, NfsCfg::NT, sm, st>>>(off, roff, V, ld_uv, core, ld_c, colour, cptr, cidx, pair_i, nidx, m_max,
                                            KA, S, vec);
    UBLR_LAUNCH_CHECK();
    dim3 gb(n_pairs, (m_max + NFB_RT - 1) / NFB_RT);
    const int nthr = (m_max + 31) / 32 * 32;
#define UBLR_NFB3(KIND, DIM)                                                                                   \
  k_nf_B3<KIND, DIM><<<gb, nthr, 0, st>>>(*op, off, roff, KA, U, ld_uv, colour, cptr, cidx, pair_i, nidx, b_off, \
                                          m_max, S, B)
    if (op->kind == UBLR_OP_LOG) {
      if (op->dim == 1) UBLR_NFB3(UBLR_OP_LOG, 1); else if (op->dim == 2) UBLR_NFB3(UBLR_OP_LOG, 2); else UBLR_NFB3(UBLR_OP_LOG, 3);
    } else {
      if (op->dim == 1) UBLR_NFB3(UBLR_OP_INV, 1); else if (op->dim == 2) UBLR_NFB3(UBLR_OP_INV, 2); else UBLR_NFB3(UBLR_OP_INV, 3);
    }
#undef UBLR_NFB3
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
  // S_p: 8 warps x NQ 8-col groups cover m_max
  int nq = (m_max + 63) / 64;  // per warp groups of 8 columns: 8 warps * 8 * nq >= m_max
#define UBLR_NFS(NA, NQ)                                                                                   \
  k_nf_S<NA, NQ><<<n_pairs, CP_THREADS, 0, st>>>(off, roff, V, ld_uv, core, ld_c, colour, cptr, cidx, pair_i, \
                                                 nidx, m_max, S)
  if (KA == 8) {
    if (nq <= 1) UBLR_NFS(1, 1); else if (nq <= 2) UBLR_NFS(1, 2); else UBLR_NFS(1, 4);
  } else if (KA == 16) {
    if (nq <= 1) UBLR_NFS(2, 1); else if (nq <= 2) UBLR_NFS(2, 2); else UBLR_NFS(2, 4);
  } else if (KA == 32) {
    if (nq <= 1) UBLR_NFS(4, 1); else if (nq <= 2) UBLR_NFS(4, 2); else UBLR_NFS(4, 4);
  } else {
    if (nq <= 1) UBLR_NFS(8, 1); else if (nq <= 2) UBLR_NFS(8, 2); else UBLR_NFS(8, 4);
  }
#undef UBLR_NFS
  UBLR_LAUNCH_CHECK();
  dim3 grid(n_pairs, (m_max + 31) / 32);
  UBLR_DISPATCH_KIND(op->kind, KIND,
                     (k_nf_B<KIND><<<grid, CP_THREADS, 0, st>>>(*op, off, roff, KA, U, ld_uv, colour, cptr, cidx,
                                                                pair_i, nidx, b_off, m_max, S, B)));
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
