// K2/K3 — sketches Y = A Omega, Z = A^* Psi with on-the-fly operator tiles.
//
// * ublr_apply: generic out = A X (every op.apply of the reference pipeline,
//   ref/operators.py:48-52): 128 x BN CTA tiles, A tile generated per k-step
//   into shared memory (k-major), X tile by cp.async, fp64 DMMA m8n8k4.
// * ublr_sketch_tagged(_pair): the tagged sketch of ref/bases.py:163-172.
//   Omega's block (j, group c) is T[j,c] G_j, so
//       Y(I_i, c*gc + q) = sum_j T[j,c] (A_ij G_j)(:, q)
//   (Kronecker restructuring): each A tile meets G_j once (2 m^2 gc flops)
//   and the ell-fold group scatter is a register epilogue per block j
//   (2 m gc ell flops) — ell times fewer flops than the dense product, with
//   every entry of Y still produced. For a symmetric operator the _pair
//   variant pushes [G | H] through one pass over A (Z = A^T Psi = A Psi).
#include "common.cuh"
#include "optile.cuh"
#include "gemm_core.cuh"
#include "tmem.cuh"
#include "ws.cuh"
#include <cstdlib>

namespace ublr {
namespace {

// ------------------------------------------------------------------ apply
constexpr int AP_BM = 128;
constexpr int AP_BK = 16;
constexpr int AP_THREADS = 256;

template <int KIND, int BN>
__global__ void __launch_bounds__(AP_THREADS) k_apply(ublr_op_t op, const double* __restrict__ X, int64_t ldx,
                                                      int w, double* __restrict__ out, int64_t ldo) {
  constexpr int SA = AP_BM + 4;
  constexpr int SB = BN + 4;
  constexpr int WN = BN / 4;        // warp tile cols (4 warps across)
  constexpr int NJ = WN / 8;        // 8-col groups per warp
  __shared__ LogTables lt;
  extern __shared__ double dsm[];
  double (*As)[AP_BK][SA] = reinterpret_cast<double (*)[AP_BK][SA]>(dsm);
  double (*Bs)[AP_BK][SB] = reinterpret_cast<double (*)[AP_BK][SB]>(dsm + 2 * AP_BK * SA);
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);

  const int n = (int)op.n;
  const int row0 = blockIdx.y * AP_BM;
  const int col0 = blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;

  // generation mapping: row = tid % 128, kk = tid / 128 + 2 i
  const int grow = tid & (AP_BM - 1);
  const int gk0 = tid >> 7;
  RowPoint rp = load_row_point(op, row0 + grow, row0 + grow < n);

  double acc[8][NJ][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  __syncthreads();  // log tables

  auto stage = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < AP_BK / 2; ++i) {
      int kk = gk0 + 2 * i;
      int q = k0 + kk;
      double v = 0.0;
      if (rp.p >= 0 && q < n) v = op_entry<KIND>(op, rp, q, &lt);
      As[buf][kk][grow] = v;
    }
    // X tile: AP_BK x BN
    for (int e = tid; e < AP_BK * BN; e += AP_THREADS) {
      int kk = e / BN, c = e - kk * BN;
      int q = k0 + kk, col = col0 + c;
      bool ok = q < n && col < w;
      cp_async8(&Bs[buf][kk][c], ok ? (const void*)(X + (int64_t)q * ldx + col) : (const void*)X, ok);
    }
    cp_async_commit();
  };

  const int nk = (n + AP_BK - 1) / AP_BK;
  stage(0, 0);
  for (int ks = 0; ks < nk; ++ks) {
    int buf = ks & 1;
    cp_async_wait<0>();
    __syncthreads();
    if (ks + 1 < nk) stage(buf ^ 1, (ks + 1) * AP_BK);
#pragma unroll
    for (int k4 = 0; k4 < AP_BK; k4 += 4) {
      double a[8], bb[NJ];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[buf][k4 + t][wr * 64 + i * 8 + g];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bb[j] = Bs[buf][k4 + t][wc * WN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int r = row0 + wr * 64 + i * 8 + g;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int c = col0 + wc * WN + j * 8 + 2 * t;
      if (c < w) out[(int64_t)r * ldo + c] = acc[i][j][0];
      if (c + 1 < w) out[(int64_t)r * ldo + c + 1] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------------ apply v2
// Producers for the shared DMMA main loop (gemm_core.cuh).
template <int KIND, class Cfg>
struct GenAProducer {
  const ublr_op_t& op;
  const LogTables* lt;
  int row0, n;
  RowPoint rp;
  int grow, gk0;
  ColRing<Cfg::BK> ring;
  __device__ GenAProducer(const ublr_op_t& op_, const LogTables* lt_, int row0_, double* ringbuf)
      : op(op_), lt(lt_), row0(row0_), n((int)op_.n) {
    grow = threadIdx.x % Cfg::BM;
    gk0 = threadIdx.x / Cfg::BM;
    rp = load_row_point(op, row0 + grow, row0 + grow < n);
    ring.buf = ringbuf;
  }
  __device__ __forceinline__ void prefetch(int ks) {
    if (KIND != UBLR_OP_DENSE) ring.prefetch(op, ks, ks * Cfg::BK, n, Cfg::NT);
  }
  __device__ __forceinline__ void stage(double* As, int ks) { stage_part(As, ks, 0, 1); }
  // entries [part*E/nparts, (part+1)*E/nparts) of this thread's E = BK/KL entries
  __device__ __forceinline__ void stage_part(double* As, int ks, int part, int nparts) {
    constexpr int KL = Cfg::NT / Cfg::BM;  // kk lanes
    constexpr int E = Cfg::BK / KL;
    const int k0 = ks * Cfg::BK;
    int e0, e1;
    chunk_range<E, 2>(part, nparts, e0, e1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e < e0 || e >= e1) continue;
      int kk = gk0 + e * KL;
      int q = k0 + kk;
      double v = 0.0;
      if (rp.p >= 0 && q < n) {
        if (KIND == UBLR_OP_DENSE) v = op_entry<KIND>(op, rp, q, lt);
        else v = kernel_entry<KIND>(op, rp, q, ring.at(ks, 0, kk), ring.at(ks, 1, kk), ring.at(ks, 2, kk), lt);
      }
      As[Cfg::ai(grow, kk)] = v;
    }
  }
};

// B tile from a row-major matrix X (K rows x N cols, ld), rows k, cols n0..
template <class Cfg>
struct RowMajorBProducer {
  const double* X;
  int64_t ld;
  int K, N, n0;
  bool vec2;
  __device__ __forceinline__ void stage(double* Bs, int ks) {
    tile_copy<Cfg::NT>(Bs, Cfg::SB, X, ld, Cfg::BK, Cfg::BN, ks * Cfg::BK, n0, K, N, IdentityRows{}, vec2);
  }
};

template <int KIND, class Cfg>
__global__ void __launch_bounds__(Cfg::NT) k_apply2(ublr_op_t op, const double* __restrict__ X, int64_t ldx, int w,
                                                    double* __restrict__ out, int64_t ldo, int vec2) {
  __shared__ LogTables lt;
  __shared__ double ringbuf[9 * Cfg::BK];
  extern __shared__ double dsm[];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int n = (int)op.n;
  const int row0 = blockIdx.x * Cfg::BM;
  const int col0 = blockIdx.y * Cfg::BN;
  GenAProducer<KIND, Cfg> ap(op, &lt, row0, ringbuf);
  RowMajorBProducer<Cfg> bp{X, ldx, n, w, col0, vec2 != 0};
  double acc[Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  __syncthreads();
  dmma_mainloop<Cfg>(ap, bp, (n + Cfg::BK - 1) / Cfg::BK, dsm, acc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int r = row0 + wr * Cfg::WM + i * 8 + g;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      int c = col0 + wc * Cfg::WN + j * 8 + 2 * t;
      if (c < w) out[(int64_t)r * ldo + c] = acc[i][j][0];
      if (c + 1 < w) out[(int64_t)r * ldo + c + 1] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------ apply, warp-specialised
// Kernel operators (A generated on the fly). Producer warps own the A tile
// (row p of the tile, a KPT-entry slice of each k-step, column points from a
// shared-memory coordinate ring) and cp.async the X tile; 8 consumer warps
// run DMMA on stages taken from a full/empty mbarrier ring, so no CTA-wide
// barrier sits inside the k loop.
//
// Why this shape (profiles/r01, tools/apply_variants.py): DMMA and the FP64
// ALU share one issue pipe. With the generation switched off the consumers
// reach 96 % of the DMMA peak; the generation costs ~22 FP64 operations per
// entry, so the tile is made wide (BN = 256: each generated entry feeds 256
// output columns) and short (BM = 64), halving the generation work per flop
// against a 128 x 128 tile. The accumulator tile (64 x 256 doubles) is what
// the register file can hold next to the fragments.
// k-steps between two flushes of the DMMA accumulators into the TMEM sums
// (0 = single-level accumulation); UBLR_APPLY_FLUSH overrides.
inline int apply_flush() {
  static const int v = [] {
    const char* e = getenv("UBLR_APPLY_FLUSH");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Second-level accumulators in tensor memory for the long k loops of the
// operator apply: the DMMA accumulators are added into TMEM every `flush`
// k-steps and restarted from zero, so a sum over n = 65,536 terms becomes
// n / (flush BK) partial sums of flush BK terms each (two-level summation:
// the rounding error of the running sum grows with the square root of the
// number of additions into one accumulator). Each consumer warp owns WD
// doubles per lane in its lane quarter; the two warps of a quarter use
// disjoint column ranges.
template <int MI, int NJ>
struct TmemAcc2 {
  static constexpr int WD = MI * NJ * 2;
  static_assert(WD % 8 == 0, "whole 8-double TMEM chunks");
  uint32_t base;
  __device__ __forceinline__ void init(uint32_t tbase, int cons_warp) {
    base = tmem::addr(tbase, cons_warp, (cons_warp >> 2) * (2 * WD));
  }
  __device__ __forceinline__ void zero() const {
    double z[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) z[q] = 0.0;
#pragma unroll
    for (int h = 0; h < WD / 8; ++h) tmem::st8(base + h * 16, z);
    tmem::wait_st();
  }
  // tm += acc; acc = 0
  __device__ __forceinline__ void flush(double (&acc)[MI][NJ][2]) const {
#pragma unroll
    for (int h0 = 0; h0 < WD / 8; h0 += 2) {
      uint32_t raw[2][16];
      tmem::ld8_async(base + h0 * 16, raw[0]);
      if (h0 + 1 < WD / 8) tmem::ld8_async(base + (h0 + 1) * 16, raw[1]);
      tmem::wait_ld();
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        if (h0 + f >= WD / 8) break;
        double v[8];
        tmem::unpack8(raw[f], v);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = (h0 + f) * 8 + q;
          v[q] += acc[e / (NJ * 2)][(e / 2) % NJ][e & 1];
          acc[e / (NJ * 2)][(e / 2) % NJ][e & 1] = 0.0;
        }
        tmem::st8(base + (h0 + f) * 16, v);
      }
    }
    tmem::wait_st();
  }
  // acc += tm
  __device__ __forceinline__ void finish(double (&acc)[MI][NJ][2]) const {
#pragma unroll
    for (int h = 0; h < WD / 8; ++h) {
      double v[8];
      tmem::ld8(base + h * 16, v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = h * 8 + q;
        acc[e / (NJ * 2)][(e / 2) % NJ][e & 1] += v[q];
      }
    }
  }
};

template <int BM_, int BN_, int BK_, int STAGES_, int WMW_, int WNW_, int NPROD_>
struct Ap3Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, WMW = WMW_, WNW = WNW_;
  static constexpr int NPROD = NPROD_, NCONS = 32 * WMW * WNW, NT = NPROD + NCONS;
  static constexpr int PH = NPROD / BM;        // producer threads per A-tile row
  static constexpr int KPT = BK / PH;          // k entries per producer thread per step
  static constexpr int PB = KPT < 8 ? KPT : 8; // entries evaluated together (ILP against the shared pipe)
  static constexpr int SA = BM + 4, SB = BN + 4;
  static constexpr int A_STAGE = BK * SA, B_STAGE = BK * SB;
  static constexpr int WM = BM / WMW, WN = BN / WNW, MI = WM / 8, NJ = WN / 8;
  // setmaxnreg moves registers inside the CTA's own pool: the kernel starts
  // at 65536 / NT (rounded down to 8) per thread; what the producers give
  // back, the consumers take.
  static constexpr int START_REGS = (65536 / NT) / 8 * 8;
  static constexpr int CONS_REGS = NT == 384 ? 208 : 200;
  static constexpr int PROD_REGS = (START_REGS * NPROD - NCONS * (CONS_REGS - START_REGS)) / NPROD / 8 * 8;
  static_assert(NPROD % BM == 0 && BK % PH == 0 && KPT % PB == 0, "producer split");
  static_assert(PROD_REGS >= 40, "producers need registers for the entry evaluation");
  static_assert(NPROD * (START_REGS - PROD_REGS) >= NCONS * (CONS_REGS - START_REGS),
                "consumers would wait forever for registers the producers never release");
  static constexpr size_t smem_bytes() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double); }
};
// Measured on B200 at c3/c4 sizes (log kernel, N = 65536, w = 4708 / 7590;
// tools/apply_variants.py): 64x256 tile, BK 16, 4 stages, 8 producer warps
// 78 / 80 % of the DMMA peak; 4 producer warps 77 / 79 %; 128x128 tile
// 71 %; the synchronous k_apply2 (UBLR_APPLY_CFG=4) 60.5 %.
using Ap3Wide = Ap3Cfg<64, 256, 16, 4, 2, 4, 256>;     // default
using Ap3Square = Ap3Cfg<128, 128, 32, 3, 2, 4, 256>;  // UBLR_APPLY_CFG=5
using Ap3Half = Ap3Cfg<64, 128, 16, 4, 2, 4, 256>;     // last column slice of <= 128 columns

template <int KIND, int DIM, class C>
__global__ void __launch_bounds__(C::NT, 1) k_apply3(ublr_op_t op, const double* __restrict__ X, int64_t ldx,
                                                     int w, double* __restrict__ out, int64_t ldo, int vec2, int flush) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::STAGES, SA = C::SA, SB = C::SB;
  constexpr int NPROD = C::NPROD, NCONS = C::NCONS, KPT = C::KPT, PB = C::PB;
  constexpr int MI = C::MI, NJ = C::NJ;
  __shared__ LogTables lt;
  __shared__ double ringbuf[9 * BK];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t tbase_slot;
  extern __shared__ double dsm[];
  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * C::A_STAGE;
  const int n = (int)op.n;
  const int row0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
  const int nk = (n + BK - 1) / BK;
  ColRing<BK> ring{ringbuf};
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ws::mbar_init(&full[s], 2 * NPROD);  // NPROD cp.async arrivals (X tile) + NPROD generator arrivals
      ws::mbar_init(&empty[s], NCONS);
    }
  }
  if (flush > 0 && threadIdx.x / 32 == NPROD / 32) tmem::alloc(&tbase_slot, 256);  // first consumer warp
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();

  if (threadIdx.x < NPROD) {
    // ---------------- producers
    ws::regs_dec<C::PROD_REGS>();
    const int p = threadIdx.x % BM;            // A-tile row
    const int kq0 = (threadIdx.x / BM) * KPT;  // first k entry of this thread
    // rows past n generate junk that is never stored; columns past n are
    // zeroed (their X rows are zero-filled too)
    const RowPoint rp = load_row_point(op, min(row0 + p, n - 1), true);
    const RowPoint rq = {row0 + p, rp.orig, rp.x0, rp.x1, rp.x2};
    const double diag = op.diag;
    ring.prefetch(op, 0, 0, n, NPROD);
    cp_async_commit();
    for (int ks = 0; ks < nk; ++ks) {
      const int s = ks % STAGES;
      const uint32_t u = (uint32_t)(ks / STAGES);
      // this step's column points: own copies landed, then every producer's
      if (ks == 0) cp_async_wait<0>();
      else cp_async_wait<1>();
      ws::named_sync(1, NPROD);
      if (ks + 1 < nk) ring.prefetch(op, ks + 1, (ks + 1) * BK, n, NPROD);
      cp_async_commit();
      ws::mbar_wait(&empty[s], (u & 1) ^ 1);
      tile_copy<NPROD>(Bs0 + s * C::B_STAGE, SB, X, ldx, BK, BN, ks * BK, col0, n, w, IdentityRows{}, vec2 != 0, 1);
      cp_async_commit();
      ws::mbar_cp_async_arrive(&full[s]);
      double* As = As0 + s * C::A_STAGE;
      const int k0 = ks * BK;
      const double* cr = ring.buf + (ks % 3) * 3 * BK;
#pragma unroll
      for (int kb = 0; kb < KPT; kb += PB) {
        double v[PB];
#pragma unroll
        for (int e = 0; e < PB; ++e) {
          const int kk = kq0 + kb + e;
          const double a = kernel_entry_dim<KIND, DIM>(rq, k0 + kk, cr[kk], DIM > 1 ? cr[BK + kk] : 0.0,
                                                       DIM > 2 ? cr[2 * BK + kk] : 0.0, diag, &lt);
          v[e] = k0 + kk < n ? a : 0.0;  // zero-filled coordinates may sit on a row point
        }
#pragma unroll
        for (int e = 0; e < PB; ++e) As[(kq0 + kb + e) * SA + p] = v[e];
      }
      ws::mbar_arrive(&full[s]);
    }
    cp_async_wait<0>();
  } else {
  // ---------------- consumers
  ws::regs_inc<C::CONS_REGS>();
  const int ct = threadIdx.x - NPROD;
  const int warp = ct >> 5, lane = ct & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / C::WNW, wc = warp % C::WNW;
  const int am0 = wr * C::WM + g, bn0 = wc * C::WN + g;
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  TmemAcc2<MI, NJ> tm;
  if (flush > 0) {
    tm.init(tbase_slot, warp);
    tm.zero();
  }
  for (int ks = 0; ks < nk; ++ks) {
    const int s = ks % STAGES;
    ws::mbar_wait(&full[s], (uint32_t)(ks / STAGES) & 1);
    const double* As = As0 + s * C::A_STAGE;
    const double* Bs = Bs0 + s * C::B_STAGE;
    double a[2][MI], b[2][NJ];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[0][i] = As[t * SA + am0 + i * 8];
#pragma unroll
    for (int j = 0; j < NJ; ++j) b[0][j] = Bs[t * SB + bn0 + j * 8];
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int cur = k4 & 1;
      if (k4 + 1 < BK / 4) {
        const int kr = (k4 + 1) * 4 + t;
#pragma unroll
        for (int i = 0; i < MI; ++i) a[cur ^ 1][i] = As[kr * SA + am0 + i * 8];
#pragma unroll
        for (int j = 0; j < NJ; ++j) b[cur ^ 1][j] = Bs[kr * SB + bn0 + j * 8];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
    }
    ws::mbar_arrive(&empty[s]);
    if (flush > 0 && (ks + 1) % flush == 0 && ks + 1 < nk) tm.flush(acc);
  }
  if (flush > 0) tm.finish(acc);
  const bool pair = (ldo % 2) == 0 && (((uintptr_t)out) % 16) == 0;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int r = row0 + wr * C::WM + i * 8 + g;
    if (r >= n) continue;
    double* orow = out + (int64_t)r * ldo;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = col0 + wc * C::WN + j * 8 + 2 * t;
      if (pair && c + 1 < w) {
        *reinterpret_cast<double2*>(orow + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < w) orow[c] = acc[i][j][0];
        if (c + 1 < w) orow[c + 1] = acc[i][j][1];
      }
    }
  }
  }
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  if (flush > 0 && threadIdx.x / 32 == NPROD / 32) tmem::dealloc(tbase_slot, 256);
}

template <class C>
int launch_apply3(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o, int vec2,
                  cudaStream_t st) {
  dim3 grid((unsigned)((op->n + C::BM - 1) / C::BM), (unsigned)((w + C::BN - 1) / C::BN));
  size_t sm = C::smem_bytes();
#define UBLR_AP3(KIND, DIM)                                                                                       \
  {                                                                                                               \
    UBLR_CUDA(cudaFuncSetAttribute(k_apply3<KIND, DIM, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_apply3<KIND, DIM, C><<<grid, C::NT, sm, st>>>(*op, X, ld_x, w, out, ld_o, vec2, apply_flush());                           \
  }
  if (op->kind == UBLR_OP_LOG) {
    if (op->dim == 1) UBLR_AP3(UBLR_OP_LOG, 1) else if (op->dim == 2) UBLR_AP3(UBLR_OP_LOG, 2) else UBLR_AP3(UBLR_OP_LOG, 3)
  } else {
    if (op->dim == 1) UBLR_AP3(UBLR_OP_INV, 1) else if (op->dim == 2) UBLR_AP3(UBLR_OP_INV, 2) else UBLR_AP3(UBLR_OP_INV, 3)
  }
#undef UBLR_AP3
  return UBLR_OK;
}

// ------------------------------- apply, warp-specialised, cluster-shared A
// k_apply3 regenerates the BM x n strip of A once per 256-column tile of X
// (18 times at c3), and that generation runs on the FP64 pipe the DMMAs need
// (ncu: DMMA 81 % + FP64 6 % of the shared pipe, the rest lost to the two
// streams interleaving). Here the CS CTAs of a thread-block cluster take
// the same row tile and CS adjacent column tiles: each generates 1/CS of
// every A stage (a BK/CS slice of the k-step) and writes it into the stage
// buffers of all CS CTAs: its own with plain stores, the peers' with
// st.async through distributed shared memory, each store signalling
// complete_tx on the peer's full[s]. Ring protocol per CTA and stage:
// full[s] collects the CTA's own X-tile cp.async arrivals, its own
// producers' arrivals (one of them expects the peers' bytes) and the
// transaction bytes of the peers' slices; empty[s] collects one arrival per
// consumer warp of every CTA (a producer overwrites the stage in all of
// them). No cluster-scope fence anywhere in the loop.
template <int KIND, int DIM, class C, int CS>
__global__ void __launch_bounds__(C::NT, 1) k_apply4(ublr_op_t op, const double* __restrict__ X, int64_t ldx,
                                                     int w, double* __restrict__ out, int64_t ldo, int vec2, int flush) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::STAGES, SA = C::SA, SB = C::SB;
  constexpr int NPROD = C::NPROD, NCONS = C::NCONS;
  constexpr int MI = C::MI, NJ = C::NJ;
  constexpr int KL = BK / CS;          // k entries of a stage generated by this CTA
  constexpr int KPT = KL / C::PH;      // ... by one producer thread
  static_assert(BK % CS == 0 && KL % C::PH == 0 && KPT >= 1, "cluster split of the k-step");
  __shared__ LogTables lt;
  __shared__ double ringbuf[9 * BK];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t tbase_slot;
  extern __shared__ double dsm[];
  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * C::A_STAGE;
  const int n = (int)op.n;
  const int row0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
  const int nk = (n + BK - 1) / BK;
  const uint32_t crank = ws::cluster_ctarank();
  ColRing<BK> ring{ringbuf};
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ws::mbar_init(&full[s], 2 * NPROD);
      ws::mbar_init(&empty[s], CS * (NCONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (flush > 0 && threadIdx.x / 32 == NPROD / 32) tmem::alloc(&tbase_slot, 256);  // first consumer warp
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  ws::cluster_sync();  // every CTA's barriers exist before a peer arrives on them

  if (threadIdx.x < NPROD) {
    // ---------------- producers
    ws::regs_dec<C::PROD_REGS>();
    const int p = threadIdx.x % BM;                              // A-tile row
    const int kq0 = (int)crank * KL + (threadIdx.x / BM) * KPT;  // first k entry of this thread
    const RowPoint rp = load_row_point(op, min(row0 + p, n - 1), true);
    const RowPoint rq = {row0 + p, rp.orig, rp.x0, rp.x1, rp.x2};
    const double diag = op.diag;
    uint32_t peer_as[CS > 1 ? CS - 1 : 1], peer_full[CS > 1 ? CS - 1 : 1];
#pragma unroll
    for (int c = 1; c < CS; ++c) {
      peer_as[c - 1] = ws::mapa(ws::smem_addr(As0), (crank + c) % CS);
      peer_full[c - 1] = ws::mapa(ws::smem_addr(&full[0]), (crank + c) % CS);
    }
    constexpr uint32_t PEER_BYTES = (uint32_t)((CS - 1) * KL * BM * sizeof(double));  // per stage, from the peers
    const bool has_cols = col0 < w;
    ring.prefetch(op, 0, 0, n, NPROD);
    cp_async_commit();
    for (int ks = 0; ks < nk; ++ks) {
      const int s = ks % STAGES;
      const uint32_t u = (uint32_t)(ks / STAGES);
      if (ks == 0) cp_async_wait<0>();
      else cp_async_wait<1>();
      ws::named_sync(1, NPROD);
      if (ks + 1 < nk) ring.prefetch(op, ks + 1, (ks + 1) * BK, n, NPROD);
      cp_async_commit();
      ws::mbar_wait(&empty[s], (u & 1) ^ 1);
      if (has_cols)
        tile_copy<NPROD>(Bs0 + s * C::B_STAGE, SB, X, ldx, BK, BN, ks * BK, col0, n, w, IdentityRows{}, vec2 != 0, 1);
      cp_async_commit();
      ws::mbar_cp_async_arrive(&full[s]);
      double* As = As0 + s * C::A_STAGE;
      const int k0 = ks * BK;
      const double* cr = ring.buf + (ks % 3) * 3 * BK;
      double v[KPT];
#pragma unroll
      for (int e = 0; e < KPT; ++e) {
        const int kk = kq0 + e;
        const double a = kernel_entry_dim<KIND, DIM>(rq, k0 + kk, cr[kk], DIM > 1 ? cr[BK + kk] : 0.0,
                                                     DIM > 2 ? cr[2 * BK + kk] : 0.0, diag, &lt);
        v[e] = k0 + kk < n ? a : 0.0;
      }
#pragma unroll
      for (int e = 0; e < KPT; ++e) {
        const int idx = s * C::A_STAGE + (kq0 + e) * SA + p;
        As0[idx] = v[e];
#pragma unroll
        for (int c = 1; c < CS; ++c)
          ws::st_async_f64(peer_as[c - 1] + (uint32_t)idx * 8u, v[e], peer_full[c - 1] + (uint32_t)s * 8u);
      }
      (void)As;
      if (CS > 1 && threadIdx.x == 0) ws::mbar_arrive_expect_tx(&full[s], PEER_BYTES);
      else ws::mbar_arrive(&full[s]);
    }
    cp_async_wait<0>();
  } else {
    // ---------------- consumers
    ws::regs_inc<C::CONS_REGS>();
    const int ct = threadIdx.x - NPROD;
    const int warp = ct >> 5, lane = ct & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = warp / C::WNW, wc = warp % C::WNW;
    const int am0 = wr * C::WM + g, bn0 = wc * C::WN + g;
    uint32_t peer_empty[CS];
#pragma unroll
    for (int c = 0; c < CS; ++c) peer_empty[c] = ws::mapa(ws::smem_addr(&empty[0]), (crank + c) % CS);
    const bool has_cols = col0 + wc * C::WN < w;   // warps past the last column skip the DMMAs
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    TmemAcc2<MI, NJ> tm;
    if (flush > 0) {
      tm.init(tbase_slot, warp);
      tm.zero();
    }
    for (int ks = 0; ks < nk; ++ks) {
      const int s = ks % STAGES;
      ws::mbar_wait(&full[s], (uint32_t)(ks / STAGES) & 1);
      if (has_cols) {
        const double* As = As0 + s * C::A_STAGE;
        const double* Bs = Bs0 + s * C::B_STAGE;
        double a[2][MI], b[2][NJ];
#pragma unroll
        for (int i = 0; i < MI; ++i) a[0][i] = As[t * SA + am0 + i * 8];
#pragma unroll
        for (int j = 0; j < NJ; ++j) b[0][j] = Bs[t * SB + bn0 + j * 8];
#pragma unroll
        for (int k4 = 0; k4 < BK / 4; ++k4) {
          const int cur = k4 & 1;
          if (k4 + 1 < BK / 4) {
            const int kr = (k4 + 1) * 4 + t;
#pragma unroll
            for (int i = 0; i < MI; ++i) a[cur ^ 1][i] = As[kr * SA + am0 + i * 8];
#pragma unroll
            for (int j = 0; j < NJ; ++j) b[cur ^ 1][j] = Bs[kr * SB + bn0 + j * 8];
          }
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
        }
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < CS; ++c) ws::mbar_arrive_remote(peer_empty[c] + (uint32_t)s * 8u);
      }
      if (flush > 0 && (ks + 1) % flush == 0 && ks + 1 < nk) tm.flush(acc);
    }
    if (flush > 0) tm.finish(acc);
    const bool pair = (ldo % 2) == 0 && (((uintptr_t)out) % 16) == 0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int r = row0 + wr * C::WM + i * 8 + g;
      if (r >= n) continue;
      double* orow = out + (int64_t)r * ldo;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = col0 + wc * C::WN + j * 8 + 2 * t;
        if (pair && c + 1 < w) {
          *reinterpret_cast<double2*>(orow + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (c < w) orow[c] = acc[i][j][0];
          if (c + 1 < w) orow[c + 1] = acc[i][j][1];
        }
      }
    }
  }
  // no CTA leaves while a peer may still store into its stages or arrive on its barriers
  tmem::fence_before();
  ws::cluster_sync();
  tmem::fence_after();
  if (flush > 0 && threadIdx.x / 32 == NPROD / 32) tmem::dealloc(tbase_slot, 256);
}

template <class C, int CS>
int launch_apply4(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o, int vec2,
                  cudaStream_t st) {
  const unsigned ty = (unsigned)((w + C::BN - 1) / C::BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((op->n + C::BM - 1) / C::BM), (ty + CS - 1) / CS * CS);
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = C::smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = CS;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define UBLR_AP4(KIND, DIM)                                                                                       \
  {                                                                                                               \
    UBLR_CUDA(cudaFuncSetAttribute(k_apply4<KIND, DIM, C, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                   (int)cfg.dynamicSmemBytes));                                                   \
    UBLR_CUDA(cudaLaunchKernelEx(&cfg, k_apply4<KIND, DIM, C, CS>, *op, X, ld_x, w, out, ld_o, vec2, apply_flush()));            \
  }
  if (op->kind == UBLR_OP_LOG) {
    if (op->dim == 1) UBLR_AP4(UBLR_OP_LOG, 1) else if (op->dim == 2) UBLR_AP4(UBLR_OP_LOG, 2) else UBLR_AP4(UBLR_OP_LOG, 3)
  } else {
    if (op->dim == 1) UBLR_AP4(UBLR_OP_INV, 1) else if (op->dim == 2) UBLR_AP4(UBLR_OP_INV, 2) else UBLR_AP4(UBLR_OP_INV, 3)
  }
#undef UBLR_AP4
  return UBLR_OK;
}

// ------------------------------------ apply through a staged strip of A
// DMMA and the FP64 ALU share one pipe, so generating A inside the GEMM costs
// tensor throughput twice: the evaluation's own pipe cycles, and the two
// instruction streams interleaving (k_apply3/4: 79-80 % of the DMMA peak,
// k_gemm3 on a stored operand: 90 %). For wide right-hand sides the strip
// form separates them in time instead of in warps: a strip of R rows of A
// (R x n doubles) is evaluated ONCE into a caller-provided HBM buffer by an
// ALU-bound kernel (every entry used to be evaluated once per 256-column
// tile: 18 times at c3, 30 at c4), then a plain k_gemm3 multiplies it by all
// w columns; the next strip reuses the buffer. A is still never stored as a
// whole (the strip is 0.5-4 GB of the 34 GB matrix at N = 65,536), the
// entries are the same bits, and the generation is ~1 % of the run.
template <int KIND, int DIM>
__global__ void __launch_bounds__(256) k_gen_strip(ublr_op_t op, int r0, int rows, double* __restrict__ out) {
  constexpr int RPC = 16;   // rows per CTA: the column point is loaded once for 16 entries
  __shared__ LogTables lt;
  __shared__ double rx[RPC][3];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int n = (int)op.n;
  const int rb = r0 + blockIdx.y * RPC;
  if (threadIdx.x < RPC * DIM) {
    const int r = threadIdx.x / DIM, d = threadIdx.x % DIM;
    rx[r][d] = rb + r < r0 + rows ? op.coords[(int64_t)d * n + rb + r] : 0.0;
  }
  __syncthreads();
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q >= n) return;
  const double c0 = op.coords[q], c1 = DIM > 1 ? op.coords[(int64_t)n + q] : 0.0,
               c2 = DIM > 2 ? op.coords[2 * (int64_t)n + q] : 0.0;
  const double diag = op.diag;
#pragma unroll 4
  for (int r = 0; r < RPC; ++r) {
    const int p = rb + r;
    if (p >= r0 + rows) break;
    const RowPoint rp = {p, 0, rx[r][0], rx[r][1], rx[r][2]};
    out[(int64_t)(p - r0) * n + q] = kernel_entry_dim<KIND, DIM>(rp, q, c0, c1, c2, diag, &lt);
  }
}

// Rows per strip: a multiple of the 128-row GEMM tile chosen so that the
// strip's CTA count (row tiles x ceil(w / 128) column tiles) fills whole
// waves of the SMs, as large as `max_bytes` allows (fewer strip boundaries).
inline int strip_rows(int64_t n, int w, int64_t max_bytes, int sms) {
  const int64_t ct = (w + 127) / 128;
  int64_t cap = max_bytes / (128 * n * 8);
  if (cap > (n + 127) / 128) cap = (n + 127) / 128;
  if (cap < 1) return 0;
  int best = 1;
  double best_eff = 0.0;
  for (int64_t rt = 1; rt <= cap; ++rt) {
    const int64_t ctas = rt * ct, waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff >= best_eff - 0.004) {   // a larger strip wins unless it wastes > 0.4 % more of its last wave
      best = (int)rt;
      if (eff > best_eff) best_eff = eff;
    }
  }
  return best * 128;
}

// ---------------------------------------------------------- tagged sketch
constexpr int TS_BM = 16;
constexpr int TS_BK = 32;
constexpr int TS_THREADS = 256;

// CTA: 16 consecutive (permuted) rows x BN of the (gc or 2gc) test-block columns.
// Warp w covers all 16 rows x BN/8 columns.
template <int KIND, int L, int BN, bool COMP = false>
__global__ void __launch_bounds__(TS_THREADS) k_sketch_tagged(ublr_op_t op, const int32_t* __restrict__ off, int b,
                                                              const double* __restrict__ T, int ell,
                                                              const double* __restrict__ G,
                                                              const double* __restrict__ H, int64_t ldx, int gc,
                                                              double* __restrict__ Y, double* __restrict__ Z,
                                                              int64_t ldy, int row_begin, int row_end) {
  constexpr int SA = TS_BM + 4;
  constexpr int SB = BN + 4;
  constexpr int WN = BN / 8;   // columns per warp
  constexpr int NJ = WN / 8;   // 8-col groups per warp
  __shared__ LogTables lt;
  extern __shared__ double dsm[];
  double (*As)[TS_BK][SA] = reinterpret_cast<double (*)[TS_BK][SA]>(dsm);
  double (*Bs)[TS_BK][SB] = reinterpret_cast<double (*)[TS_BK][SB]>(dsm + 2 * TS_BK * SA);
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);

  const int ncols = (H ? 2 : 1) * gc;
  // rows are independent in the sketch, so 16-row tiles may straddle blocks
  const int rend = row_end;
  const int row0 = row_begin + blockIdx.y * TS_BM;
  const int col0 = blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  const int grow = tid & (TS_BM - 1);
  const int gk0 = tid >> 4;  // 0..15; entries kk = gk0, gk0 + 16
  RowPoint rp = load_row_point(op, row0 + grow, row0 + grow < rend);

  double acc[L][2][NJ][2];
#pragma unroll
  for (int c = 0; c < L; ++c)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[c][r][j][0] = acc[c][r][j][1] = 0.0;
  double wacc[2][NJ][2];
  // COMP: compensated fold (the rounding error of every acc += tc * w is
  // recovered exactly with an error-free product and TwoSum, and summed apart)
  double cacc[COMP ? L : 1][2][NJ][2];
#pragma unroll
  for (int c = 0; c < (COMP ? L : 1); ++c)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < NJ; ++j) cacc[c][r][j][0] = cacc[c][r][j][1] = 0.0;

  __syncthreads();

  auto stage = [&](int buf, int q0, int qend) {
#pragma unroll
    for (int e = 0; e < TS_BK / 16; ++e) {
      int kk = gk0 + 16 * e;
      int q = q0 + kk;
      double v = 0.0;
      if (rp.p >= 0 && q < qend) v = op_entry<KIND>(op, rp, q, &lt);
      As[buf][kk][grow] = v;
    }
    for (int e = tid; e < TS_BK * BN; e += TS_THREADS) {
      int kk = e / BN, c = e - kk * BN;
      int q = q0 + kk, col = col0 + c;
      bool ok = q < qend && col < ncols;
      const double* src = G;
      if (ok) src = (col < gc) ? (G + (int64_t)q * ldx + col) : (H + (int64_t)q * ldx + (col - gc));
      cp_async8(&Bs[buf][kk][c], src, ok);
    }
    cp_async_commit();
  };

  // flattened (block j, k-step) loop
  int j = 0, q0 = off[0];
  int qend = off[1];
  stage(0, q0, qend);
  int buf = 0;
  for (;;) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) wacc[r][jj][0] = wacc[r][jj][1] = 0.0;
    for (;;) {
      // next stage coordinates
      int nq0 = q0 + TS_BK, nj = j, nqend = qend;
      if (nq0 >= qend) {
        nj = j + 1;
        if (nj < b) { nq0 = off[nj]; nqend = off[nj + 1]; }
      }
      cp_async_wait<0>();
      __syncthreads();
      if (nj < b) stage(buf ^ 1, nq0, nqend);
#pragma unroll
      for (int k4 = 0; k4 < TS_BK; k4 += 4) {
        double a0 = As[buf][k4 + t][g];
        double a1 = As[buf][k4 + t][8 + g];
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
          double bb = Bs[buf][k4 + t][warp * WN + jj * 8 + g];
          mma8x8x4(wacc[0][jj][0], wacc[0][jj][1], a0, bb);
          mma8x8x4(wacc[1][jj][0], wacc[1][jj][1], a1, bb);
        }
      }
      buf ^= 1;
      bool block_done = (nj != j);
      q0 = nq0; qend = nqend;
      if (block_done) break;
    }
    // scatter block j's product into the ell tag groups
#pragma unroll
    for (int c = 0; c < L; ++c) {
      double tc = (c < ell) ? __ldg(&T[(int64_t)j * ell + c]) : 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
          if (COMP) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double a = acc[c][r][jj][h], w = wacc[r][jj][h];
              const double pr = tc * w, pe = fma(tc, w, -pr);
              const double sm = a + pr, bb = sm - a;
              const double e = (a - (sm - bb)) + (pr - bb);
              cacc[COMP ? c : 0][r][jj][h] += e + pe;
              acc[c][r][jj][h] = sm;
            }
          } else {
            acc[c][r][jj][0] = fma(tc, wacc[r][jj][0], acc[c][r][jj][0]);
            acc[c][r][jj][1] = fma(tc, wacc[r][jj][1], acc[c][r][jj][1]);
          }
        }
    }
    ++j;
    if (j >= b) break;
  }
  // epilogue: (row, col) -> Y or Z at group c
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    int row = row0 + r * 8 + g;
    if (row >= rend) continue;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int col = col0 + warp * WN + jj * 8 + 2 * t + h;
        if (col >= ncols) continue;
        double* dst = (col < gc) ? Y : Z;
        int q = (col < gc) ? col : col - gc;
#pragma unroll
        for (int c = 0; c < L; ++c)
          if (c < ell) dst[(int64_t)row * ldy + c * gc + q] = acc[c][r][jj][h] + (COMP ? cacc[COMP ? c : 0][r][jj][h] : 0.0);
      }
  }
}

// ------------------------------------------------------- tagged sketch v3
// CTA = BM (32) permuted rows x BN (128 or 64) test-block columns, 8 warps
// (2 x 4; warp tile 16 x BN/4). The ell tag-group accumulators of the CTA
// (BM x BN x ell doubles: 320 KB for 32 x 128 x 10) do not fit in the
// register file, so the first TG groups live in TMEM (tcgen05.st/ld, 256 KB
// per SM) and the rest in registers. Every A tile is generated once per
// (row tile, column tile) — once per row tile when 2gc <= BN — and every
// test-block panel is reused by BM rows.
template <int KIND, int L, class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1) k_sketch_tagged3(ublr_op_t op_a, const int32_t* __restrict__ off, int b,
                                                               const double* __restrict__ T, int ell,
                                                               const double* __restrict__ G,
                                                               const double* __restrict__ H, int64_t ldx, int gc,
                                                               double* __restrict__ Y, double* __restrict__ Z,
                                                               int64_t ldy, int row_begin, int row_end, int vec2,
                                                               ublr_op_t op_b, const double* __restrict__ G_b,
                                                               double* __restrict__ Y_b) {
  // gridDim.z == 2: blockIdx.z = 1 sketches a second operator (the adjoint of a
  // non-symmetric A) against its own test blocks in the same launch
  const ublr_op_t op = blockIdx.z ? op_b : op_a;
  if (blockIdx.z) {
    G = G_b;
    Y = Y_b;
  }
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int WD = Cfg::MI * Cfg::NJ * 2;            // W doubles per thread
  constexpr int NWARP = Cfg::NT / 32;
  constexpr int WCOLS = 512 / (NWARP / 4);             // TMEM columns per warp (warps sharing a lane quarter split 512)
  constexpr int WDP = (WD + 7) / 8 * 8;                // TMEM stride per group (whole x16 chunks)
  constexpr int TCAP = (WCOLS / 2) / WDP;              // groups per thread that fit
  constexpr int TG = (L < TCAP) ? L : TCAP;            // groups kept in TMEM
  constexpr int RG = L - TG;                           // groups kept in registers
  static_assert(NWARP % 4 == 0, "lane quarters are shared evenly");
  static_assert(TG * WDP * 2 <= WCOLS, "TMEM groups overflow the warp's columns");
  __shared__ LogTables lt;
  __shared__ uint32_t tbase_slot;
  extern __shared__ double dsm[];
  if (KIND == UBLR_OP_LOG) init_log_tables(&lt);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (warp == 0) tmem::alloc(&tbase_slot, 512);
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  const uint32_t tbase = tbase_slot;
  const int colbase = (warp >> 2) * WCOLS;           // warps sharing a lane quarter split its columns

  const int ncols = (H ? 2 : 1) * gc;
  const int row0 = row_begin + blockIdx.x * Cfg::BM;
  const int col0 = blockIdx.y * Cfg::BN;
  // A producer (absolute columns q0.. masked by qend), interleavable
  __shared__ double ringbuf[9 * BK];
  struct AP {
    const ublr_op_t& op; const LogTables* lt; RowPoint rp; int grow, gk0;
    int q0n, qendn;   // columns of the stage being produced
    int sidx;         // its stage index (ring slot)
    ColRing<BK> ring;
    // dense, not transposed: thread = (column kk, rows dr[e]) so a warp reads
    // consecutive columns of one row of A (coalesced); dorig[e] = perm[row] or -1
    int dorig[(BK * Cfg::BM + Cfg::NT - 1) / Cfg::NT];
    __device__ __forceinline__ void stage_part(double* As, int, int part, int nparts) {
      constexpr int KL = Cfg::NT / Cfg::BM;
      constexpr int E = BK / KL;
      int e0, e1;
      chunk_range<E, 2>(part, nparts, e0, e1);
      if (KIND == UBLR_OP_DENSE && !op.transpose) {
        static_assert(BK * Cfg::BM % Cfg::NT == 0 && Cfg::NT % BK == 0, "dense tile mapping");
        const int kk = threadIdx.x % BK;
        const int q = q0n + kk;
        const bool qok = q < qendn;
        const int oq = qok ? (op.perm ? op.perm[q] : q) : 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e < e0 || e >= e1) continue;
          const int rr = threadIdx.x / BK + e * (Cfg::NT / BK);
          const double v = (qok && dorig[e] >= 0) ? op.A[(int64_t)dorig[e] * op.lda + oq] : 0.0;
          As[Cfg::ai(rr, kk)] = v;
        }
        return;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e < e0 || e >= e1) continue;
        int kk = gk0 + e * KL;
        int q = q0n + kk;
        double v = 0.0;
        if (rp.p >= 0 && q < qendn) {
          if (KIND == UBLR_OP_DENSE) v = op_entry<KIND>(op, rp, q, lt);
          else v = kernel_entry<KIND>(op, rp, q, ring.at(sidx, 0, kk), ring.at(sidx, 1, kk), ring.at(sidx, 2, kk), lt);
        }
        As[Cfg::ai(grow, kk)] = v;
      }
    }
  } ap{op, &lt, load_row_point(op, row0 + (int)(threadIdx.x % Cfg::BM), row0 + (int)(threadIdx.x % Cfg::BM) < row_end),
       (int)(threadIdx.x % Cfg::BM), (int)(threadIdx.x / Cfg::BM), 0, 0, 0, ColRing<BK>{ringbuf}, {}};
  if (KIND == UBLR_OP_DENSE) {
#pragma unroll
    for (int e = 0; e < (int)(sizeof(ap.dorig) / sizeof(int)); ++e) {
      const int row = row0 + (int)(threadIdx.x / BK) + e * (Cfg::NT / BK);
      ap.dorig[e] = row < row_end ? (op.perm ? op.perm[row] : row) : -1;
    }
  }
  // test-block panel stage: BK rows x BN columns of [G | H]. Each thread's
  // 16-byte pair slots are fixed for the whole kernel, so their source
  // pointers (minus the k-step row offset) are computed once here.
  constexpr int HALF = Cfg::BN / 2;
  constexpr int PPT = (BK * HALF + Cfg::NT - 1) / Cfg::NT;
  const bool vec_pairs = vec2 != 0 && (gc % 2) == 0;
  const double* bsrc[PPT];
  int bmeta[PPT];  // smem offset | kk << 16 | (column valid) << 30
#pragma unroll
  for (int z = 0; z < PPT; ++z) {
    const int e = threadIdx.x + z * Cfg::NT;
    const int kk = e / HALF, c = 2 * (e % HALF);
    const int col = col0 + c;
    const bool valid = e < BK * HALF && col < ncols;
    bsrc[z] = ((col < gc || !H) ? G + col : H + (col - gc)) + (int64_t)kk * ldx;
    bmeta[z] = (kk * Cfg::SB + c) | (kk << 16) | (valid ? (1 << 30) : 0);
  }
  auto b_stage = [&](double* Bs, int q0, int qend) {
    if (vec_pairs) {
      const int64_t roff = (int64_t)q0 * ldx;
#pragma unroll
      for (int z = 0; z < PPT; ++z) {
        const int meta = bmeta[z];
        const bool ok = (meta >> 30) && q0 + ((meta >> 16) & 0x3fff) < qend;
        cp_async16(Bs + (meta & 0xffff), ok ? (const void*)(bsrc[z] + roff) : (const void*)G, ok);
      }
    } else if (col0 + Cfg::BN <= gc || !H) {
      tile_copy<Cfg::NT>(Bs, Cfg::SB, G, ldx, BK, Cfg::BN, q0, col0, qend, gc, IdentityRows{}, vec2 != 0);
    } else if (col0 >= gc) {
      tile_copy<Cfg::NT>(Bs, Cfg::SB, H, ldx, BK, Cfg::BN, q0, col0 - gc, qend, gc, IdentityRows{}, vec2 != 0);
    } else {
      for (int e = threadIdx.x; e < BK * Cfg::BN; e += Cfg::NT) {
        int kk = e / Cfg::BN, c = e - kk * Cfg::BN;
        int q = q0 + kk, col = col0 + c;
        bool ok = q < qend && col < ncols;
        const double* src = G;
        if (ok) src = (col < gc) ? (G + (int64_t)q * ldx + col) : (H + (int64_t)q * ldx + (col - gc));
        cp_async8(&Bs[kk * Cfg::SB + c], src, ok);
      }
    }
  };

  double w[Cfg::MI][Cfg::NJ][2];
  double racc[RG > 0 ? RG : 1][Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      w[i][j][0] = w[i][j][1] = 0.0;
#pragma unroll
      for (int c = 0; c < (RG > 0 ? RG : 1); ++c) racc[c][i][j][0] = racc[c][i][j][1] = 0.0;
    }
  {  // zero the TMEM groups
    double z[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) z[q] = 0.0;
#pragma unroll
    for (int c = 0; c < TG; ++c)
#pragma unroll
      for (int h = 0; h < WDP / 8; ++h) tmem::st8(tmem::addr(tbase, warp, colbase + (c * WDP + h * 8) * 2), z);
    tmem::wait_st();
  }
  __syncthreads();

  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * Cfg::A_STAGE;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
  const int am0 = wr * Cfg::WM + g;
  const int bn0 = wc * Cfg::WN + g;
  // stage coordinates: (block, first column, end column); advance() walks k-steps block by block
  auto advance = [&](int& jj, int& qq0, int& qqe) {
    qq0 += BK;
    if (qq0 >= qqe) {
      ++jj;
      if (jj < b) { qq0 = off[jj]; qqe = off[jj + 1]; }
    }
  };
  int j = 0, q0 = off[0], qend = off[1];
  int j1 = j, q01 = q0, qe1 = qend;
  advance(j1, q01, qe1);
  if (KIND != UBLR_OP_DENSE) {
    ap.ring.prefetch(op, 0, q0, qend, Cfg::NT);
    if (j1 < b) ap.ring.prefetch(op, 1, q01, qe1, Cfg::NT);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  ap.q0n = q0; ap.qendn = qend; ap.sidx = 0;
  ap.stage_part(As0, 0, 0, 1);
  b_stage(Bs0, q0, qend);
  cp_async_commit();
  int slot = 0, sidx = 0;
  for (;;) {
    // next stage (j1, q01, qe1) and the one after (j2, q02, qe2)
    int nj = j1, nq0 = q01, nqend = qe1;
    int j2 = nj, q02 = nq0, qe2 = nqend;
    if (nj < b) advance(j2, q02, qe2);
    const bool more = nj < b;
    cp_async_wait<0>();
    __syncthreads();
    double* As_nx = As0 + (slot ^ 1) * Cfg::A_STAGE;
    if (more) b_stage(Bs0 + (slot ^ 1) * Cfg::B_STAGE, nq0, nqend);
    if (KIND != UBLR_OP_DENSE && more && j2 < b) ap.ring.prefetch(op, sidx + 2, q02, qe2, Cfg::NT);
    ap.q0n = nq0; ap.qendn = nqend; ap.sidx = sidx + 1;
    const double* As = As0 + slot * Cfg::A_STAGE;
    const double* Bs = Bs0 + slot * Cfg::B_STAGE;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int kr = k4 * 4 + t;
      double a[Cfg::MI], bb[Cfg::NJ];
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i) a[i] = As[Cfg::ai(am0 + i * 8, kr)];
#pragma unroll
      for (int jj = 0; jj < Cfg::NJ; ++jj) bb[jj] = Bs[Cfg::bi(kr, bn0 + jj * 8)];
      if (more) ap.stage_part(As_nx, 0, k4, BK / 4);
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int jj = 0; jj < Cfg::NJ; ++jj) mma8x8x4(w[i][jj][0], w[i][jj][1], a[i], bb[jj]);
    }
    cp_async_commit();
    if (nj != j) {
      // block j complete: acc_c += T[j, c] * W  (TMEM groups, then register groups)
      const double* Tj = T + (int64_t)j * ell;
      double wf[WDP];
#pragma unroll
      for (int q = WD; q < WDP; ++q) wf[q] = 0.0;
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int jj = 0; jj < Cfg::NJ; ++jj) {
          wf[(i * Cfg::NJ + jj) * 2] = w[i][jj][0];
          wf[(i * Cfg::NJ + jj) * 2 + 1] = w[i][jj][1];
          w[i][jj][0] = w[i][jj][1] = 0.0;
        }
#pragma unroll
      for (int c = 0; c < TG; ++c) {
        const double tc = (c < ell) ? __ldg(&Tj[c]) : 0.0;
#pragma unroll
        for (int h = 0; h < WDP / 8; ++h) {
          double v[8];
          const uint32_t ta = tmem::addr(tbase, warp, colbase + (c * WDP + h * 8) * 2);
          tmem::ld8(ta, v);
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = fma(tc, wf[h * 8 + q], v[q]);
          tmem::st8(ta, v);
        }
      }
#pragma unroll
      for (int c = 0; c < RG; ++c) {
        const double tc = (TG + c < ell) ? __ldg(&Tj[TG + c]) : 0.0;
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
          for (int jj = 0; jj < Cfg::NJ; ++jj) {
            racc[c][i][jj][0] = fma(tc, wf[(i * Cfg::NJ + jj) * 2], racc[c][i][jj][0]);
            racc[c][i][jj][1] = fma(tc, wf[(i * Cfg::NJ + jj) * 2 + 1], racc[c][i][jj][1]);
          }
      }
      tmem::wait_st();
    }
    if (!more) break;
    j = nj; q0 = nq0; qend = nqend;
    j1 = j2; q01 = q02; qe1 = qe2;
    slot ^= 1;
    ++sidx;
  }
  cp_async_wait<0>();
  // epilogue
#pragma unroll
  for (int c = 0; c < L; ++c) {
    if (c >= ell) break;
    double accv[WDP];
    if (c < TG) {
#pragma unroll
      for (int h = 0; h < WDP / 8; ++h) {
        double v[8];
        tmem::ld8(tmem::addr(tbase, warp, colbase + (c * WDP + h * 8) * 2), v);
#pragma unroll
        for (int q = 0; q < 8; ++q) accv[h * 8 + q] = v[q];
      }
    } else {
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int jj = 0; jj < Cfg::NJ; ++jj) {
          accv[(i * Cfg::NJ + jj) * 2] = racc[(c - TG) < 0 ? 0 : (c - TG)][i][jj][0];
          accv[(i * Cfg::NJ + jj) * 2 + 1] = racc[(c - TG) < 0 ? 0 : (c - TG)][i][jj][1];
        }
    }
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i) {
      int row = row0 + wr * Cfg::WM + i * 8 + g;
      if (row >= row_end) continue;
#pragma unroll
      for (int jj = 0; jj < Cfg::NJ; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int col = col0 + wc * Cfg::WN + jj * 8 + 2 * t + h;
          if (col >= ncols) continue;
          double* dst = (col < gc) ? Y : Z;
          int q = (col < gc) ? col : col - gc;
          dst[(int64_t)row * ldy + c * gc + q] = accv[(i * Cfg::NJ + jj) * 2 + h];
        }
    }
  }
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  if (warp == 0) tmem::dealloc(tbase, 512);
}


// ------------------------------------------------- tagged sketch v4 (warp-specialised)
// Same product as v3 (Y(I, c gc + q) = sum_j T[j,c] (A_Ij G_j)(:, q), both
// sides) with the roles split: 8 producer warps generate the BM x BK A tile
// (kernel operators) and cp.async the BK x BN [G | H] panel into a STAGES-deep
// full/empty mbarrier ring; 8 consumer warps (2 x 4, warp tile 16 x BN/4) run
// the DMMAs and, after the last k-step of every block j, fold W into the ell
// tag groups (TG of them in TMEM, the rest in registers). Producers run ahead
// across block boundaries while the consumers fold.
template <int BN_, int STAGES_>
struct Sk4Cfg {
  static constexpr int BM = 32, BN = BN_, BK = 16, STAGES = STAGES_;
  static constexpr int NPROD = 256, NCONS = 256, NT = NPROD + NCONS;
  static constexpr int WMW = 2, WNW = 4, WM = BM / WMW, WN = BN / WNW, MI = WM / 8, NJ = WN / 8;
  static constexpr int SA = BM + 4, SB = BN + 4;
  static constexpr int SAM = BK + 4;   // STAGED: the A stage is copied m-major (As[m][k], as its source is stored)
  static constexpr int A_STAGE = BK * SA > BM * SAM ? BK * SA : BM * SAM, B_STAGE = BK * SB;
  static constexpr int CONS_REGS = 200, PROD_REGS = 56;
  static constexpr size_t smem_bytes() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double); }
  // compensated fold: 16 bytes (8 bf16 error sums) per consumer thread and 8-entry chunk of each tag group
  static constexpr int WD = MI * NJ * 2, WDP = (WD + 7) / 8 * 8;
  static constexpr int TCAP = ((512 / (NCONS / 32 / 4)) / 2) / WDP;   // tag groups a warp's TMEM columns hold
  static constexpr size_t comp_bytes(int L) { return (size_t)NCONS * 16 * (size_t)(L * (WDP / 8)); }
};

// Compensated fold (COMP). Z_c = sum_j T[j,c] W_j adds b = 256 increments of
// size ~|W_j| into an accumulator of size ~sqrt(b)|W_j|: its rounding errors
// (one per fold, half an ulp of the running sum) are the largest noise term
// of the tagged sketch, and type B divides the pair-combined sketch by
// projected tags as small as 1e-4 and pushes it through the core least
// squares, so that noise IS the approximation error of B2 at N = 65,536
// (measured: 9.1e-9 -> 5.4e-9 with the errors recovered; reference 7.1e-9).
// Per fold s = fma(t, w, a) is followed by e = fma(t, w, a - s), the exact
// error when |t w| <~ |a| (a - s is then exact), and e is summed apart: in
// bf16 in shared memory for the TMEM groups (TMEM is full; |sum e| is a few
// ulp(a), so 8 mantissa bits leave ~0.1 ulp), in fp32 registers for the
// register groups; the epilogue adds the error sums to the accumulators.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// STAGED: the rows [strip_r0, ...) of A have been evaluated into `strip`
// (row-major, ld = n) by k_gen_strip, and the producers only copy: A tiles
// with 16-byte cp.async into an m-major stage, next to the panel. No FP64
// work competes with the DMMAs (the evaluation inside the kernel holds the
// DMMA pipe at 43-57 %: the consumers own the pipe while they have a stage,
// the producers' chains advance when they wait), and A is evaluated once per
// strip instead of once per column tile. Needs n and every off[j] even.
template <int KIND, int DIM, int L, class C, bool COMP = false, bool STAGED = false>
__global__ void __launch_bounds__(C::NT, 1) k_sketch_tagged4(ublr_op_t op, const int32_t* __restrict__ off, int b,
                                                             const double* __restrict__ T, int ell,
                                                             const double* __restrict__ G,
                                                             const double* __restrict__ H, int64_t ldx, int gc,
                                                             double* __restrict__ Y, double* __restrict__ Z,
                                                             int64_t ldy, int row_begin, int row_end,
                                                             const double* __restrict__ strip = nullptr,
                                                             int strip_r0 = 0) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::STAGES, SA = C::SA, SB = C::SB;
  constexpr int MI = C::MI, NJ = C::NJ;
  constexpr int WD = MI * NJ * 2;                       // W doubles per consumer thread
  constexpr int WCOLS = 512 / (C::NCONS / 32 / 4);      // TMEM columns per consumer warp
  constexpr int WDP = (WD + 7) / 8 * 8;
  constexpr int TCAP = (WCOLS / 2) / WDP;
  constexpr int TG = (L < TCAP) ? L : TCAP;
  constexpr int RG = L - TG;
  __shared__ LogTables lt;
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t tbase_slot;
  extern __shared__ double dsm[];
  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * C::A_STAGE;
  uint4* comp = reinterpret_cast<uint4*>(dsm + STAGES * (C::A_STAGE + C::B_STAGE));  // COMP: [chunk][consumer thread]
  const int ncols = (H ? 2 : 1) * gc;
  const int row0 = row_begin + blockIdx.x * BM;
  const int col0 = blockIdx.y * BN;
  const int n = (int)op.n;
  if (KIND == UBLR_OP_LOG && !STAGED) init_log_tables(&lt);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // arrivals per stage: one cp.async arrival per producer thread (its
      // panel copies have landed) + one per producer warp (its A entries are
      // stored) on full; one per consumer warp on empty. An mbarrier takes
      // arrivals one at a time, so per-thread arrivals (768 per stage) cost
      // more than the stage's DMMAs
      ws::mbar_init(&full[s], C::NPROD + C::NPROD / 32);
      ws::mbar_init(&empty[s], C::NCONS / 32);
    }
  }
  if (threadIdx.x / 32 == C::NPROD / 32) tmem::alloc(&tbase_slot, 512);  // first consumer warp
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  const uint32_t tbase = tbase_slot;

  if (threadIdx.x < C::NPROD) {
    // ---------------- producers
    ws::regs_dec<C::PROD_REGS>();
    const int p = threadIdx.x;
    const int r = p % BM;               // A-tile row
    const int kq = p / BM;              // k lane (BM x BK / NPROD = 2 entries per thread: kq, kq + 8)
    constexpr int KL = C::NPROD / BM;
    constexpr int EPT = BK / KL;
    const bool rok = row0 + r < row_end;
    const RowPoint rp = load_row_point(op, rok ? row0 + r : row_begin, true);
    const double diag = op.diag;
    // panel pair slots, fixed for the kernel (see v3)
    constexpr int HALF = BN / 2;
    constexpr int PPT = (BK * HALF + C::NPROD - 1) / C::NPROD;
    const double* bsrc[PPT];
    int bmeta[PPT];
#pragma unroll
    for (int z = 0; z < PPT; ++z) {
      const int e = p + z * C::NPROD;
      const int kk = e / HALF, c = 2 * (e % HALF);
      const int col = col0 + c;
      const bool valid = e < BK * HALF && col < ncols;
      bsrc[z] = ((col < gc || !H) ? G + col : H + (col - gc)) + (int64_t)kk * ldx;
      bmeta[z] = (kk * SB + c) | (kk << 16) | (valid ? (1 << 30) : 0);
    }
    int it = 0;
    if (STAGED) {
      // copy-only producers: thread p moves the 16-byte pair (row p / 8, k pair p % 8) of the A tile
      static_assert(!STAGED || (C::NPROD == BM * BK / 2), "one 16-byte A chunk per producer thread");
      const int pr = p >> 3, pk2 = (p & 7) * 2;
      const int prow = row0 + pr < row_end ? row0 + pr : row_begin;      // rows past the end: any valid row
      const double* arow = strip + (int64_t)(prow - strip_r0) * n;
      for (int j = 0; j < b; ++j) {
        const int qe = off[j + 1];
        for (int q0 = off[j]; q0 < qe; q0 += BK, ++it) {
          const int s = it % STAGES;
          ws::mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1) ^ 1);
          double* Bs = Bs0 + s * C::B_STAGE;
          const int64_t roff = (int64_t)q0 * ldx;
#pragma unroll
          for (int z = 0; z < PPT; ++z) {
            const int meta = bmeta[z];
            const bool ok = (meta >> 30) && q0 + ((meta >> 16) & 0x3fff) < qe;
            cp_async16(Bs + (meta & 0xffff), ok ? (const void*)(bsrc[z] + roff) : (const void*)G, ok);
          }
          double* Ad = As0 + s * C::A_STAGE + pr * C::SAM + pk2;
          const int k = q0 + pk2;
          if (k + 1 < qe) {
            cp_async16(Ad, arow + k, true);
          } else {                       // the k dimension ends inside this pair: zeros past the end
            cp_async8(Ad, k < qe ? (const void*)(arow + k) : (const void*)strip, k < qe);
            cp_async8(Ad + 1, strip, false);
          }
          cp_async_commit();
          ws::mbar_cp_async_arrive(&full[s]);
          __syncwarp();
          if ((p & 31) == 0) ws::mbar_arrive(&full[s]);
        }
      }
      cp_async_wait<0>();
    } else {
    // column coordinates are loaded one stage ahead (software pipelining: the
    // global-load latency of stage it + 1 hides behind the evaluations of it)
    double cn[EPT][DIM];
    auto load_cols = [&](int q0, int qe) {
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int q = q0 + kq + e * KL;
        const int qc = q < qe ? q : q0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) cn[e][d] = __ldg(op.coords + (int64_t)d * n + qc);
      }
    };
    load_cols(off[0], off[1]);
    for (int j = 0; j < b; ++j) {
      const int qe = off[j + 1];
      for (int q0 = off[j]; q0 < qe; q0 += BK, ++it) {
        const int s = it % STAGES;
        double cc[EPT][DIM];
#pragma unroll
        for (int e = 0; e < EPT; ++e)
#pragma unroll
          for (int d = 0; d < DIM; ++d) cc[e][d] = cn[e][d];
        if (q0 + BK < qe) load_cols(q0 + BK, qe);
        else if (j + 1 < b) load_cols(qe, off[j + 2]);
        double v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const int q = q0 + kq + e * KL;
          const bool ok = q < qe;
          const int qc = ok ? q : q0;
          const double a = kernel_entry_dim<KIND, DIM>(rp, qc, cc[e][0], DIM > 1 ? cc[e][DIM > 1 ? 1 : 0] : 0.0,
                                                       DIM > 2 ? cc[e][DIM > 2 ? 2 : 0] : 0.0, diag, &lt);
          v[e] = ok ? a : 0.0;
        }
        ws::mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1) ^ 1);
        double* Bs = Bs0 + s * C::B_STAGE;
        const int64_t roff = (int64_t)q0 * ldx;
#pragma unroll
        for (int z = 0; z < PPT; ++z) {
          const int meta = bmeta[z];
          const bool ok = (meta >> 30) && q0 + ((meta >> 16) & 0x3fff) < qe;
          cp_async16(Bs + (meta & 0xffff), ok ? (const void*)(bsrc[z] + roff) : (const void*)G, ok);
        }
        cp_async_commit();
        ws::mbar_cp_async_arrive(&full[s]);
        double* As = As0 + s * C::A_STAGE;
#pragma unroll
        for (int e = 0; e < EPT; ++e) As[(kq + e * KL) * SA + r] = v[e];
        __syncwarp();
        if ((p & 31) == 0) ws::mbar_arrive(&full[s]);
      }
    }
    cp_async_wait<0>();
    }
  } else {
    // ---------------- consumers
    ws::regs_inc<C::CONS_REGS>();
    const int ct = threadIdx.x - C::NPROD;
    const int warp = ct >> 5, lane = ct & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = warp / C::WNW, wc = warp % C::WNW;
    const int am0 = wr * C::WM + g, bn0 = wc * C::WN + g;
    const int twarp = warp;                       // lane quarter = warp & 3
    const int colbase = (warp >> 2) * WCOLS;
    // 8-column groups of this warp's slice that hold columns of [G | H]: the
    // last column tile is mostly padding (c4: 20 of 128 columns), and its
    // DMMAs on zero-filled panel columns would cost what real ones do
    const int ncol_w = ncols - (col0 + wc * C::WN);
    const int nj_valid = ncol_w <= 0 ? 0 : (ncol_w >= C::WN ? NJ : (ncol_w + 7) / 8);
    double w[MI][NJ][2];
    double racc[RG > 0 ? RG : 1][MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        w[i][jj][0] = w[i][jj][1] = 0.0;
#pragma unroll
        for (int c = 0; c < (RG > 0 ? RG : 1); ++c) racc[c][i][jj][0] = racc[c][i][jj][1] = 0.0;
      }
    if (COMP) {
#pragma unroll
      for (int ch = 0; ch < L * (WDP / 8); ++ch) comp[ch * C::NCONS + ct] = make_uint4(0u, 0u, 0u, 0u);
    }
    {
      double z8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) z8[q] = 0.0;
#pragma unroll
      for (int c = 0; c < TG; ++c)
#pragma unroll
        for (int h = 0; h < WDP / 8; ++h) tmem::st8(tmem::addr(tbase, twarp, colbase + (c * WDP + h * 8) * 2), z8);
      tmem::wait_st();
    }
    int it = 0;
    for (int j = 0; j < b; ++j) {
      const int qe = off[j + 1];
      for (int q0 = off[j]; q0 < qe; q0 += BK, ++it) {
        const int s = it % STAGES;
        ws::mbar_wait(&full[s], (uint32_t)(it / STAGES) & 1);
        const double* As = As0 + s * C::A_STAGE;
        const double* Bs = Bs0 + s * C::B_STAGE;
        static_assert(MI == 2, "the m16n8k8 fragments cover the warp's two 8-row blocks");
        // m16n8k8 DMMA: a0..a3 = A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4];
        // b0, b1 = B[t][g], B[t+4][g]; d = (w[0][jj], w[1][jj]) -- the m8n8k4 layout
        if (nj_valid == NJ) {
          // m8n8k4 DMMAs (16 pipe cycles each instead of 64 for m16n8k8): the
          // producers' FP64 evaluations get a slot between two of them four
          // times as often (c5 shard sketch 1573 -> 1473 ms; c4 unchanged)
#pragma unroll
          for (int k4 = 0; k4 < BK / 4; ++k4) {
            const int kr = k4 * 4 + t;
            const double a0 = STAGED ? As[am0 * C::SAM + kr] : As[kr * SA + am0];
            const double a1 = STAGED ? As[(am0 + 8) * C::SAM + kr] : As[kr * SA + am0 + 8];
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
              const double b0 = Bs[kr * SB + bn0 + jj * 8];
              mma8x8x4(w[0][jj][0], w[0][jj][1], a0, b0);
              mma8x8x4(w[1][jj][0], w[1][jj][1], a1, b0);
            }
          }
        } else if (nj_valid > 0) {   // last column tile: only the 8-column groups that hold columns
#pragma unroll
          for (int k8 = 0; k8 < BK / 8; ++k8) {
            const int kr = k8 * 8 + t;
            const double a0 = STAGED ? As[am0 * C::SAM + kr] : As[kr * SA + am0];
            const double a1 = STAGED ? As[(am0 + 8) * C::SAM + kr] : As[kr * SA + am0 + 8];
            const double a2 = STAGED ? As[am0 * C::SAM + kr + 4] : As[(kr + 4) * SA + am0];
            const double a3 = STAGED ? As[(am0 + 8) * C::SAM + kr + 4] : As[(kr + 4) * SA + am0 + 8];
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
              if (jj < nj_valid) {
                const double b0 = Bs[kr * SB + bn0 + jj * 8], b1 = Bs[(kr + 4) * SB + bn0 + jj * 8];
                mma16x8x8(w[0][jj][0], w[0][jj][1], w[1][jj][0], w[1][jj][1], a0, a1, a2, a3, b0, b1);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) ws::mbar_arrive(&empty[s]);
      }
      if (nj_valid == 0) continue;   // a warp past the last column has nothing to fold
      // block j complete: acc_c += T[j, c] W
      const double* Tj = T + (int64_t)j * ell;
      double wf[WDP];
#pragma unroll
      for (int q = WD; q < WDP; ++q) wf[q] = 0.0;
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
          wf[(i * NJ + jj) * 2] = w[i][jj][0];
          wf[(i * NJ + jj) * 2 + 1] = w[i][jj][1];
          w[i][jj][0] = w[i][jj][1] = 0.0;
        }
      // TMEM groups in batches of FB chunks: issue the loads, one wait, FMAs, stores
      constexpr int NCH = TG * (WDP / 8);           // 8-double chunks held in TMEM
      constexpr int FB = COMP ? 1 : (NCH < (WDP > 8 ? 2 : 4) ? NCH : (WDP > 8 ? 2 : 4));
#pragma unroll
      for (int c0 = 0; c0 < NCH; c0 += FB) {
        uint32_t raw[FB][16];
#pragma unroll
        for (int f = 0; f < FB; ++f)
          if (c0 + f < NCH) tmem::ld8_async(tmem::addr(tbase, twarp, colbase + (c0 + f) * 16), raw[f]);
        tmem::wait_ld();
#pragma unroll
        for (int f = 0; f < FB; ++f) {
          if (c0 + f >= NCH) break;
          const int c = (c0 + f) / (WDP / 8), h = (c0 + f) % (WDP / 8);
          const double tc = (c < ell) ? __ldg(&Tj[c]) : 0.0;
          double v[8];
          tmem::unpack8(raw[f], v);
          if (COMP) {
            uint4* cp = comp + (c0 + f) * C::NCONS + ct;
            const uint4 cb = *cp;
            const uint32_t cw[4] = {cb.x, cb.y, cb.z, cb.w};
            uint32_t nw[4];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              float e2[2] = {__uint_as_float(cw[q2] << 16), __uint_as_float(cw[q2] & 0xffff0000u)};
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int q = 2 * q2 + hh;
                const double a = v[q], ww = wf[h * 8 + q];
                const double sm = fma(tc, ww, a);
                e2[hh] += __double2float_rn(fma(tc, ww, a - sm));
                v[q] = sm;
              }
              nw[q2] = pack_bf16x2(e2[0], e2[1]);
            }
            *cp = make_uint4(nw[0], nw[1], nw[2], nw[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = fma(tc, wf[h * 8 + q], v[q]);
          }
          tmem::st8(tmem::addr(tbase, twarp, colbase + (c0 + f) * 16), v);
        }
      }
#pragma unroll
      for (int c = 0; c < RG; ++c) {
        const double tc = (TG + c < ell) ? __ldg(&Tj[TG + c]) : 0.0;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj) {
            if (!COMP) {
              racc[c][i][jj][0] = fma(tc, wf[(i * NJ + jj) * 2], racc[c][i][jj][0]);
              racc[c][i][jj][1] = fma(tc, wf[(i * NJ + jj) * 2 + 1], racc[c][i][jj][1]);
            }
          }
        if (COMP) {
#pragma unroll
          for (int h = 0; h < WDP / 8; ++h) {
            uint4* cp = comp + ((TG + c) * (WDP / 8) + h) * C::NCONS + ct;
            const uint4 cb = *cp;
            const uint32_t cw[4] = {cb.x, cb.y, cb.z, cb.w};
            uint32_t nw[4];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              float e2[2] = {__uint_as_float(cw[q2] << 16), __uint_as_float(cw[q2] & 0xffff0000u)};
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int e = h * 8 + 2 * q2 + hh;
                if (e < WD) {
                  double& a = racc[c][e / (NJ * 2)][(e / 2) % NJ][e & 1];
                  const double ww = wf[e];
                  const double sm = fma(tc, ww, a);
                  e2[hh] += __double2float_rn(fma(tc, ww, a - sm));
                  a = sm;
                }
              }
              nw[q2] = pack_bf16x2(e2[0], e2[1]);
            }
            *cp = make_uint4(nw[0], nw[1], nw[2], nw[3]);
          }
        }
      }
    }
    tmem::wait_st();
    // epilogue: Y / Z rows of this warp
#pragma unroll
    for (int c = 0; c < L; ++c) {
      if (c >= ell) break;
      double accv[WDP];
      if (c < TG) {
#pragma unroll
        for (int h = 0; h < WDP / 8; ++h) {
          double v[8];
          tmem::ld8(tmem::addr(tbase, twarp, colbase + (c * WDP + h * 8) * 2), v);
          if (COMP) {
            const uint4 cb = comp[(c * (WDP / 8) + h) * C::NCONS + ct];
            const uint32_t cw[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              v[2 * q2] += (double)__uint_as_float(cw[q2] << 16);
              v[2 * q2 + 1] += (double)__uint_as_float(cw[q2] & 0xffff0000u);
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) accv[h * 8 + q] = v[q];
        }
      } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj) {
            accv[(i * NJ + jj) * 2] = racc[(c - TG) < 0 ? 0 : (c - TG)][i][jj][0];
            accv[(i * NJ + jj) * 2 + 1] = racc[(c - TG) < 0 ? 0 : (c - TG)][i][jj][1];
          }
        if (COMP) {
#pragma unroll
          for (int h = 0; h < WDP / 8; ++h) {
            const uint4 cb = comp[(c * (WDP / 8) + h) * C::NCONS + ct];
            const uint32_t cw[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              accv[h * 8 + 2 * q2] += (double)__uint_as_float(cw[q2] << 16);
              accv[h * 8 + 2 * q2 + 1] += (double)__uint_as_float(cw[q2] & 0xffff0000u);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = row0 + wr * C::WM + i * 8 + g;
        if (row >= row_end) continue;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = col0 + wc * C::WN + jj * 8 + 2 * t + h;
            if (col >= ncols) continue;
            double* dst = (col < gc) ? Y : Z;
            const int q = (col < gc) ? col : col - gc;
            dst[(int64_t)row * ldy + c * gc + q] = accv[(i * NJ + jj) * 2 + h];
          }
      }
    }
  }
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  if (threadIdx.x / 32 == C::NPROD / 32) tmem::dealloc(tbase, 512);
}
}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_apply(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o,
                          void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(w >= 0 && X && out && ld_x >= w && ld_o >= w, UBLR_ERR_VALUE, "ublr_apply: bad X/out");
  if (w == 0) return UBLR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid;
  using CfgW = TileCfg<128, 128, 32, 4, 4, 2>;
  using CfgN = TileCfg<128, 64, 32, 4, 4, 2>;
  static int variant = [] {
    const char* e = getenv("UBLR_APPLY_CFG");
    return e ? atoi(e) : 0;
  }();
  int vec2 = ((ld_x % 2) == 0 && (((uintptr_t)X) % 16) == 0) ? 1 : 0;
  // row tiles fastest (grid.x): CTAs in flight share one X column slab in L2
#define UBLR_AP2(CFG)                                                                                         \
  UBLR_DISPATCH_KIND(op->kind, KIND, {                                                                      \
    grid.x = (unsigned)((op->n + CFG::BM - 1) / CFG::BM);                                                   \
    grid.y = (unsigned)((w + CFG::BN - 1) / CFG::BN);                                                       \
    size_t sm = CFG::smem_bytes();                                                                          \
    UBLR_CUDA(cudaFuncSetAttribute(k_apply2<KIND, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_apply2<KIND, CFG><<<grid, CFG::NT, sm, st>>>(*op, X, ld_x, w, out, ld_o, vec2);                         \
  })
  if (w > 64 && op->kind != UBLR_OP_DENSE && variant == 5) {
    rc = launch_apply3<Ap3Square>(op, X, ld_x, w, out, ld_o, vec2, st);
    if (rc) return rc;
  } else if (w > 64 && op->kind != UBLR_OP_DENSE && variant == 0) {
    // column ranges: clusters of 2 CTAs sharing the generated A strip over
    // whole pairs of 256-column tiles, the remainder on single CTAs (a
    // 128-column tile for a last slice of <= 128 columns). All offsets are
    // multiples of 256 columns, so the 16-byte alignment of X / out carries
    // over. Measured on B200 (N = 65,536, w = 4096): single CTAs 79.4 %,
    // 2-CTA clusters 80.1 %; clusters of 4 51 % (a 4-CTA cluster strands 16 of
    // the 148 SMs) and are not built. UBLR_APPLY_CS=1 turns clusters off.
    // Also measured and dropped: fetching the next stage's first fragments
    // during a stage's last k4 slice (test_wait one slice early): 78.5 %.
    static const int cs_max = [] {
      const char* e = getenv("UBLR_APPLY_CS");
      return e ? atoi(e) : 2;
    }();
    int c0 = 0;
    if (cs_max >= 2 && (w - c0) >= 2 * Ap3Wide::BN) {
      const int wm = (w - c0) / (2 * Ap3Wide::BN) * (2 * Ap3Wide::BN);
      rc = launch_apply4<Ap3Wide, 2>(op, X + c0, ld_x, wm, out + c0, ld_o, vec2, st);
      if (rc) return rc;
      c0 += wm;
    }
    int rem = w - c0;
    if (rem > 0) {
      int wfull = rem / Ap3Wide::BN * Ap3Wide::BN;
      if (rem - wfull > Ap3Half::BN) wfull = rem;
      if (wfull > 0) {
        rc = launch_apply3<Ap3Wide>(op, X + c0, ld_x, wfull, out + c0, ld_o, vec2, st);
        if (rc) return rc;
        c0 += wfull;
      }
      if (w - c0 > 0) {
        rc = launch_apply3<Ap3Half>(op, X + c0, ld_x, w - c0, out + c0, ld_o, vec2, st);
        if (rc) return rc;
      }
    }
  } else if (w <= 64) {
    UBLR_AP2(CfgN);
  } else {
    UBLR_AP2(CfgW);  // dense operator, or UBLR_APPLY_CFG=4 (the synchronous k_apply2)
  }
#undef UBLR_AP2
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

namespace {
// v1: 16-row tiles (kept as default: measured faster than v2 on c2/c4 shapes, profiles/r01)
int sketch_common_v1(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell, const double* G,
                     const double* H, int64_t ld_x, int gc, double* Y, double* Z, int64_t ld_y, int row_begin,
                     int row_end, cudaStream_t st, bool comp = false) {
  int ncols = (H ? 2 : 1) * gc;
  dim3 grid;
  grid.y = (unsigned)((row_end - row_begin + TS_BM - 1) / TS_BM);
#define UBLR_TS_LAUNCH(L, BN)                                                                              \
  {                                                                                                        \
    grid.x = (unsigned)((ncols + (BN) - 1) / (BN));                                                       \
    UBLR_DISPATCH_KIND(op->kind, KIND, {                                                                  \
      size_t sm = (size_t)2 * TS_BK * ((TS_BM + 4) + ((BN) + 4)) * sizeof(double);                       \
      UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged<KIND, L, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)sm));                                                          \
      k_sketch_tagged<KIND, L, BN><<<grid, TS_THREADS, sm, st>>>(*op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, \
                                                                 row_begin, row_end);                  \
    })                                                                                                     \
  }
  if (ell <= 4 && !comp) UBLR_TS_LAUNCH(4, 128)
  else if (ell <= 10 && comp) {
    grid.x = (unsigned)((ncols + 63) / 64);
    UBLR_DISPATCH_KIND(op->kind, KIND, {
      size_t sm = (size_t)2 * TS_BK * ((TS_BM + 4) + (64 + 4)) * sizeof(double);
      UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged<KIND, 10, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
      k_sketch_tagged<KIND, 10, 64, true><<<grid, TS_THREADS, sm, st>>>(*op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y,
                                                                        row_begin, row_end);
    })
  }
  else if (ell <= 10) UBLR_TS_LAUNCH(10, 64)
  else if (ell <= 28) UBLR_TS_LAUNCH(28, 64)
  else {
    set_error("tagged sketch supports ell <= 28 (d <= 3 without extra columns)");
    return UBLR_ERR_VALUE;
  }
#undef UBLR_TS_LAUNCH
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

int sketch_common_v3(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell, const double* G,
                     const double* H, int64_t ld_x, int gc, double* Y, double* Z, int64_t ld_y, int row_begin,
                     int row_end, cudaStream_t st, const ublr_op_t* op2 = nullptr, const double* G2 = nullptr,
                     double* Y2 = nullptr) {
  const int ncols = (H ? 2 : 1) * gc;
  int vec2 = ((ld_x % 2) == 0 && ((uintptr_t)G) % 16 == 0 && (!H || ((uintptr_t)H) % 16 == 0) &&
              (!G2 || ((uintptr_t)G2) % 16 == 0)) ? 1 : 0;
  dim3 grid;
  grid.z = op2 ? 2 : 1;
  const ublr_op_t opb = op2 ? *op2 : *op;
  static const int ts_cfg = [] {
    const char* e = getenv("UBLR_SKETCH_CFG");
    return e ? atoi(e) : 0;
  }();
#define UBLR_TS3(L, BNv)                                                                                        \
  { if (ts_cfg == 1 && (BNv) == 128) {                                                                          \
    using Cfg = TileCfg<32, BNv, 32, 2, 4, 2>;                                                                  \
    UBLR_TS3_LAUNCH(L)                                                                                          \
  } else if (ts_cfg == 2 && (BNv) == 128) {                                                                     \
    using Cfg = TileCfg<32, BNv, 32, 2, 4, 3>;                                                                  \
    UBLR_TS3_LAUNCH(L)                                                                                          \
  } else {                                                                                                      \
    using Cfg = TileCfg<32, BNv, 32, 2, 8, 2>;                                                                  \
    UBLR_TS3_LAUNCH(L)                                                                                          \
  } }
#define UBLR_TS3_LAUNCH(L)                                                                                      \
  {                                                                                                             \
    grid.y = (unsigned)((ncols + Cfg::BN - 1) / Cfg::BN);                                                        \
    grid.x = (unsigned)((row_end - row_begin + 31) / 32);                                                       \
    UBLR_DISPATCH_KIND(op->kind, KIND, {                                                                        \
      size_t sm = Cfg::smem_bytes();                                                                            \
      UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged3<KIND, L, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)sm));                                                                \
      k_sketch_tagged3<KIND, L, Cfg><<<grid, Cfg::NT, sm, st>>>(*op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y,   \
                                                                row_begin, row_end, vec2, opb, G2, Y2);        \
    })                                                                                                          \
  }
  if (ncols <= 64) {
    if (ell <= 4) UBLR_TS3(4, 64) else UBLR_TS3(10, 64)
  } else {
    if (ell <= 4) UBLR_TS3(4, 128) else UBLR_TS3(10, 128)
  }
#undef UBLR_TS3
#undef UBLR_TS3_LAUNCH
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

int sketch_common_v4(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell, const double* G,
                     const double* H, int64_t ld_x, int gc, double* Y, double* Z, int64_t ld_y, int row_begin,
                     int row_end, cudaStream_t st, bool comp = false) {
  const int ncols = (H ? 2 : 1) * gc;
  dim3 grid((unsigned)((row_end - row_begin + 31) / 32), 0);
#define UBLR_TS4(KIND, DIM, L, BNv)                                                                              \
  {                                                                                                              \
    using C = Sk4Cfg<BNv, 6>;                                                                                    \
    grid.y = (unsigned)((ncols + C::BN - 1) / C::BN);                                                            \
    size_t sm = C::smem_bytes();                                                                                 \
    UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged4<KIND, DIM, L, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   (int)sm));                                                                   \
    k_sketch_tagged4<KIND, DIM, L, C><<<grid, C::NT, sm, st>>>(*op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y,   \
                                                               row_begin, row_end);                              \
  }
  // (measured no faster on B200 and dropped: a 96-column tile for c4's 532
  // columns — 6 x 96 = 576 padded columns instead of 5 x 128 = 640 — 266.6 vs
  // 262.7 ms, the sixth regeneration of the A tile costs what the padding
  // saved; BK = 32 with 4 stages — c4 278 vs 263 ms, c5 shard 1662 vs
  // 1573 ms, the 56-register producers spill)
#define UBLR_TS4_L(KIND, DIM)                                                                                    \
  {                                                                                                              \
    if (ncols <= 64) {                                                                                           \
      if (ell <= 4) UBLR_TS4(KIND, DIM, 4, 64) else UBLR_TS4(KIND, DIM, 10, 64)                                  \
    } else {                                                                                                     \
      if (ell <= 4) UBLR_TS4(KIND, DIM, 4, 128) else UBLR_TS4(KIND, DIM, 10, 128)                                \
    }                                                                                                            \
  }
#define UBLR_TS4C(KIND, DIM)                                                                                     \
  {                                                                                                              \
    using C = Sk4Cfg<128, 6>;                                                                                    \
    grid.y = (unsigned)((ncols + C::BN - 1) / C::BN);                                                            \
    size_t sm = C::smem_bytes() + C::comp_bytes(10);                                                             \
    UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged4<KIND, DIM, 10, C, true>,                                     \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                      \
    k_sketch_tagged4<KIND, DIM, 10, C, true><<<grid, C::NT, sm, st>>>(*op, off, b, T, ell, G, H, ld_x, gc, Y, Z,  \
                                                                      ld_y, row_begin, row_end);                 \
  }
  if (comp) {   // compensated fold (type B): one tile shape, ell <= 10
    if (op->kind == UBLR_OP_LOG) {
      if (op->dim == 1) UBLR_TS4C(UBLR_OP_LOG, 1) else if (op->dim == 2) UBLR_TS4C(UBLR_OP_LOG, 2) else UBLR_TS4C(UBLR_OP_LOG, 3)
    } else {
      if (op->dim == 1) UBLR_TS4C(UBLR_OP_INV, 1) else if (op->dim == 2) UBLR_TS4C(UBLR_OP_INV, 2) else UBLR_TS4C(UBLR_OP_INV, 3)
    }
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
#undef UBLR_TS4C
  if (op->kind == UBLR_OP_LOG) {
    if (op->dim == 1) UBLR_TS4_L(UBLR_OP_LOG, 1) else if (op->dim == 2) UBLR_TS4_L(UBLR_OP_LOG, 2) else UBLR_TS4_L(UBLR_OP_LOG, 3)
  } else {
    if (op->dim == 1) UBLR_TS4_L(UBLR_OP_INV, 1) else if (op->dim == 2) UBLR_TS4_L(UBLR_OP_INV, 2) else UBLR_TS4_L(UBLR_OP_INV, 3)
  }
#undef UBLR_TS4_L
#undef UBLR_TS4
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

// Rows per strip of the staged tagged sketch: a multiple of the 32-row tile
// such that rt x ct CTAs (ct column tiles) fill whole waves of the SMs; 0 if
// no strip within `max_bytes` reaches 85 % of its last wave (a c5 shard has one
// column tile: 148 row tiles = 4,736 rows = 40 GB of strip at N = 2^20).
inline int sketch_strip_rows(int64_t n, int ncols, int64_t rows_total, int64_t max_bytes, int sms,
                             bool require_eff = true) {
  const int64_t ct = (ncols + (ncols <= 64 ? 63 : 127)) / (ncols <= 64 ? 64 : 128);
  int64_t cap = max_bytes / (32 * n * 8);
  if (cap > (rows_total + 31) / 32) cap = (rows_total + 31) / 32;
  int best = 0;
  double best_eff = 0.0;
  for (int64_t rt = 1; rt <= cap; ++rt) {
    const int64_t ctas = rt * ct, waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff >= best_eff - 0.004) {
      best = (int)rt;
      if (eff > best_eff) best_eff = eff;
    }
  }
  if (!require_eff) return best * 32;                                            // the entry point runs with any strip
  if (cap >= (rows_total + 31) / 32 && best_eff < 0.85) return (int)cap * 32;   // the whole range fits: one strip
  return best_eff >= 0.85 ? best * 32 : 0;
}

int sketch_staged(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell, const double* G,
                  const double* H, int64_t ld_x, int gc, double* Y, double* Z, int64_t ld_y, int row_begin,
                  int row_end, bool comp, double* strip, int R, cudaStream_t st) {
  const int ncols = (H ? 2 : 1) * gc;
  const int64_t n = op->n;
  for (int r0 = row_begin; r0 < row_end; r0 += R) {
    const int r1 = r0 + R < row_end ? r0 + R : row_end;
    dim3 ggrid((unsigned)((n + 255) / 256), (unsigned)((r1 - r0 + 15) / 16));
#define UBLR_GEN(KIND, DIM) k_gen_strip<KIND, DIM><<<ggrid, 256, 0, st>>>(*op, r0, r1 - r0, strip)
    if (op->kind == UBLR_OP_LOG) {
      if (op->dim == 1) UBLR_GEN(UBLR_OP_LOG, 1); else if (op->dim == 2) UBLR_GEN(UBLR_OP_LOG, 2); else UBLR_GEN(UBLR_OP_LOG, 3);
    } else {
      if (op->dim == 1) UBLR_GEN(UBLR_OP_INV, 1); else if (op->dim == 2) UBLR_GEN(UBLR_OP_INV, 2); else UBLR_GEN(UBLR_OP_INV, 3);
    }
#undef UBLR_GEN
    UBLR_LAUNCH_CHECK();
    dim3 grid((unsigned)((r1 - r0 + 31) / 32), 0);
#define UBLR_TS5(L, BNv, COMPv)                                                                                  \
  {                                                                                                              \
    using C = Sk4Cfg<BNv, 6>;                                                                                    \
    grid.y = (unsigned)((ncols + C::BN - 1) / C::BN);                                                            \
    size_t sm = C::smem_bytes() + ((COMPv) ? C::comp_bytes(10) : 0);                                             \
    UBLR_CUDA(cudaFuncSetAttribute(k_sketch_tagged4<UBLR_OP_INV, 1, L, C, COMPv, true>,                          \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                      \
    k_sketch_tagged4<UBLR_OP_INV, 1, L, C, COMPv, true><<<grid, C::NT, sm, st>>>(                                \
        *op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, r0, r1, strip, r0);                                     \
  }
    if (comp) UBLR_TS5(10, 128, true)
    else if (ncols <= 64) { if (ell <= 4) UBLR_TS5(4, 64, false) else UBLR_TS5(10, 64, false) }
    else { if (ell <= 4) UBLR_TS5(4, 128, false) else UBLR_TS5(10, 128, false) }
#undef UBLR_TS5
    UBLR_LAUNCH_CHECK();
  }
  return UBLR_OK;
}

int sketch_common(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell, const double* G,
                  const double* H, int64_t ld_x, int gc, double* Y, double* Z, int64_t ld_y, int row_begin,
                  int row_end, cudaStream_t st, bool comp = false) {
  UBLR_REQUIRE(row_begin >= 0 && row_begin < row_end && row_end <= op->n, UBLR_ERR_VALUE, "sketch: bad row range");
  if (comp && ell <= 10) {
    // compensated fold: the warp-specialised kernel for kernel operators, the
    // 16-row register-tile kernel otherwise (dense A, unaligned panels)
    const bool vok = (ld_x % 2) == 0 && (gc % 2) == 0 && ((uintptr_t)G) % 16 == 0 && (!H || ((uintptr_t)H) % 16 == 0);
    if ((op->kind == UBLR_OP_LOG || op->kind == UBLR_OP_INV) && vok)
      return sketch_common_v4(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, st, true);
    return sketch_common_v1(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, st, true);
  }
  static const char* ver = getenv("UBLR_SKETCH_VERSION");
  const int v = ver ? atoi(ver) : 4;
  const bool vec_ok = (ld_x % 2) == 0 && (gc % 2) == 0 && ((uintptr_t)G) % 16 == 0 && (!H || ((uintptr_t)H) % 16 == 0);
  // v4 (warp-specialised): c2 0.246 -> 0.196 ms, c4 325 -> 263 ms (table log);
  // c5 shard 1.98 -> 1.57 s (1/r)
  // 1/r: v4 since its m16n8k8 consumers and one-stage-ahead column loads
  // (c5 shard 1.98 s with v3 -> 1.57 s); UBLR_SKETCH_V4_INV=0 restores v3
  static const bool v4_inv = [] {
    const char* e = getenv("UBLR_SKETCH_V4_INV");
    return !e || atoi(e) != 0;
  }();
  if (v == 4 && ell <= 10 && (op->kind == UBLR_OP_LOG || (v4_inv && op->kind == UBLR_OP_INV)) && vec_ok)
    return sketch_common_v4(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, st);
  if (v >= 3 && ell <= 10) return sketch_common_v3(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, st);
  return sketch_common_v1(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, st);
}

}  // namespace

extern "C" int ublr_sketch_tagged(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                                  const double* X, int64_t ld_x, int gc, double* Y, int64_t ld_y, int row_begin,
                                  int row_end, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && T && X && Y && gc > 0 && ell > 0 && ld_x >= gc && ld_y >= (int64_t)ell * gc,
               UBLR_ERR_VALUE, "ublr_sketch_tagged: bad arguments");
  return sketch_common(op, off, b, T, ell, X, nullptr, ld_x, gc, Y, nullptr, ld_y, row_begin, row_end,
                       (cudaStream_t)stream);
}

extern "C" int ublr_sketch_tagged_two(const ublr_op_t* op, const ublr_op_t* op_adj, const int32_t* off, int b,
                                      const double* T, int ell, const double* G, const double* H, int64_t ld_x, int gc,
                                      double* Y, double* Z, int64_t ld_y, int row_begin, int row_end, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  rc = check_op(op_adj);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && T && G && H && Y && Z && gc > 0 && ell > 0 && ld_x >= gc &&
                   ld_y >= (int64_t)ell * gc && op->kind == op_adj->kind && op->n == op_adj->n,
               UBLR_ERR_VALUE, "ublr_sketch_tagged_two: bad arguments");
  UBLR_REQUIRE(row_begin >= 0 && row_begin < row_end && row_end <= op->n, UBLR_ERR_VALUE, "sketch: bad row range");
  cudaStream_t st = (cudaStream_t)stream;
  static const char* ver = getenv("UBLR_SKETCH_VERSION");
  const int v = ver ? atoi(ver) : 4;
  if (v >= 3 && ell <= 10)
    return sketch_common_v3(op, off, b, T, ell, G, nullptr, ld_x, gc, Y, nullptr, ld_y, row_begin, row_end, st,
                            op_adj, H, Z);
  rc = sketch_common(op, off, b, T, ell, G, nullptr, ld_x, gc, Y, nullptr, ld_y, row_begin, row_end, st);
  if (rc) return rc;
  return sketch_common(op_adj, off, b, T, ell, H, nullptr, ld_x, gc, Z, nullptr, ld_y, row_begin, row_end, st);
}

extern "C" int ublr_sketch_tagged_pair(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                                       const double* G, const double* H, int64_t ld_x, int gc, double* Y, double* Z,
                                       int64_t ld_y, int row_begin, int row_end, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && T && G && H && Y && Z && gc > 0 && ell > 0 && ld_x >= gc &&
                   ld_y >= (int64_t)ell * gc,
               UBLR_ERR_VALUE, "ublr_sketch_tagged_pair: bad arguments");
  return sketch_common(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, (cudaStream_t)stream);
}

extern "C" int ublr_sketch_tagged_comp(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                                       const double* G, const double* H, int64_t ld_x, int gc, double* Y, double* Z,
                                       int64_t ld_y, int row_begin, int row_end, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && T && G && Y && (!H == !Z) && gc > 0 && ell > 0 && ld_x >= gc &&
                   ld_y >= (int64_t)ell * gc,
               UBLR_ERR_VALUE, "ublr_sketch_tagged_comp: bad arguments");
  return sketch_common(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, (cudaStream_t)stream,
                       true);
}

// Largest strip the staged apply asks for (it runs with any workspace of at
// least one 128-row strip).
extern "C" int64_t ublr_apply_staged_workspace_bytes(int64_t n, int w) {
  const int64_t want = (int64_t)4 << 30;
  const int rows = strip_rows(n, w, want, 148);
  return (int64_t)(rows > 0 ? rows : 128) * n * 8;
}

static int device_sms() {
  static const int sms = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

// Rows per strip the staged apply uses with a workspace of this size (0: too small).
extern "C" int ublr_apply_staged_rows(int64_t n, int w, int64_t workspace_bytes) {
  return strip_rows(n, w, workspace_bytes, device_sms());
}

extern "C" int ublr_apply_staged(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o,
                                 void* workspace, int64_t workspace_bytes, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(w >= 0 && X && out && ld_x >= w && ld_o >= w, UBLR_ERR_VALUE, "ublr_apply_staged: bad X/out");
  UBLR_REQUIRE(op->kind == UBLR_OP_LOG || op->kind == UBLR_OP_INV, UBLR_ERR_VALUE,
               "ublr_apply_staged: kernel operators only (a dense A is already stored)");
  if (w == 0) return UBLR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = op->n;
  const int R = strip_rows(n, w, workspace_bytes, device_sms());
  UBLR_REQUIRE(workspace && R >= 128, UBLR_ERR_VALUE, "ublr_apply_staged: workspace smaller than one 128-row strip");
  double* strip = (double*)workspace;
  for (int64_t r0 = 0; r0 < n; r0 += R) {
    const int rows = (int)(n - r0 < R ? n - r0 : R);
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)((rows + 15) / 16));
#define UBLR_GEN(KIND, DIM) k_gen_strip<KIND, DIM><<<grid, 256, 0, st>>>(*op, (int)r0, rows, strip)
    if (op->kind == UBLR_OP_LOG) {
      if (op->dim == 1) UBLR_GEN(UBLR_OP_LOG, 1); else if (op->dim == 2) UBLR_GEN(UBLR_OP_LOG, 2); else UBLR_GEN(UBLR_OP_LOG, 3);
    } else {
      if (op->dim == 1) UBLR_GEN(UBLR_OP_INV, 1); else if (op->dim == 2) UBLR_GEN(UBLR_OP_INV, 2); else UBLR_GEN(UBLR_OP_INV, 3);
    }
#undef UBLR_GEN
    UBLR_LAUNCH_CHECK();
    rc = ublr_gemm_batched(0, 0, rows, w, (int)n, 1.0, strip, n, 0, nullptr, 0, X, ld_x, 0, nullptr, 0, 0.0,
                           out + r0 * ld_o, ld_o, 0, nullptr, 0, 1, stream);
    if (rc) return rc;
  }
  return UBLR_OK;
}

// Rows per strip of ublr_sketch_tagged_staged with this workspace (0: no
// strip of that size keeps the SMs busy -- use the fused entry points).
extern "C" int ublr_sketch_tagged_staged_rows(int64_t n, int ncols, int rows, int64_t workspace_bytes) {
  return sketch_strip_rows(n, ncols, rows, workspace_bytes, device_sms());
}

extern "C" int ublr_sketch_tagged_staged(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                                         const double* G, const double* H, int64_t ld_x, int gc, double* Y, double* Z,
                                         int64_t ld_y, int row_begin, int row_end, int compensated, void* workspace,
                                         int64_t workspace_bytes, void* stream) {
  int rc = check_op(op);
  if (rc) return rc;
  UBLR_REQUIRE(b > 0 && off && T && G && Y && (!H == !Z) && gc > 0 && ell > 0 && ell <= 10 && ld_x >= gc &&
                   ld_y >= (int64_t)ell * gc && row_begin >= 0 && row_begin < row_end && row_end <= op->n,
               UBLR_ERR_VALUE, "ublr_sketch_tagged_staged: bad arguments (ell <= 10)");
  UBLR_REQUIRE((op->kind == UBLR_OP_LOG || op->kind == UBLR_OP_INV) && op->n % 2 == 0, UBLR_ERR_VALUE,
               "ublr_sketch_tagged_staged: kernel operators with an even number of points");
  UBLR_REQUIRE((ld_x % 2) == 0 && (gc % 2) == 0 && ((uintptr_t)G) % 16 == 0 && (!H || ((uintptr_t)H) % 16 == 0) &&
                   workspace && ((uintptr_t)workspace) % 16 == 0,
               UBLR_ERR_VALUE, "ublr_sketch_tagged_staged: 16-byte aligned panels and workspace, even gc / ld_x");
  const int ncols = (H ? 2 : 1) * gc;
  const int R = sketch_strip_rows(op->n, ncols, row_end - row_begin, workspace_bytes, device_sms(), false);
  UBLR_REQUIRE(R >= 32, UBLR_ERR_VALUE, "ublr_sketch_tagged_staged: workspace smaller than one 32-row strip");
  return sketch_staged(op, off, b, T, ell, G, H, ld_x, gc, Y, Z, ld_y, row_begin, row_end, compensated != 0,
                       (double*)workspace, R, (cudaStream_t)stream);
}
