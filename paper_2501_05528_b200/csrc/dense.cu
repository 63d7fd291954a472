// Batched dense fp64 building blocks for the block-nullification and type-B
// solves (no cuBLAS/cuSOLVER on the hot path):
//
// * ublr_gemm_batched: C_b = alpha op(A_b) op(B_b) + beta C_b, row-major,
//   optional storage-row gather maps (so Omega[nbr(i)] is read in place, no
//   stacked copy), fp64 DMMA m8n8k4, 128x128 / 64x64 CTA tiles.
// * ublr_potrf_diag: Cholesky (upper, A = R^T R) of an nb x nb diagonal block
//   per batch entry in shared memory, plus R^-1 — the panel step of a
//   right-looking blocked Cholesky driven from the host (dense.py).
// * ublr_lu_sign_diag: LU without pivoting of an nb x nb diagonal block with
//   the Householder-reconstruction sign choice (Ballard et al.): before each
//   pivot j, D_jj = -sign(w_jj) is added to the diagonal, so |pivot| >= 1.
//   Applied to D - Q1_top this reproduces LAPACK's dlarfg reflectors
//   (tau_j = pivot_j * D_jj in [1, 2]); see DESIGN.md §bn null space.
//   Also returns L^-1 and U^-1 of the block.
#include "common.cuh"
#include "gemm_core.cuh"
#include "ws.cuh"

namespace ublr {
namespace {

constexpr int GT = 256;
constexpr int GBK = 16;

template <class Cfg, bool TA, bool TB>
__global__ void __launch_bounds__(Cfg::NT) k_gemm2(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                   int64_t lda, int64_t sA, const int32_t* __restrict__ amap,
                                                   int64_t sAm, const double* __restrict__ B, int64_t ldb, int64_t sB,
                                                   const int32_t* __restrict__ bmap, int64_t sBm, double beta,
                                                   double* __restrict__ C, int64_t ldc, int64_t sC,
                                                   const int32_t* __restrict__ cmap, int64_t sCm, int vecA, int vecB,
                                                   int upper_only) {
  static_assert(Cfg::A_KM == TA && Cfg::B_KM == !TB, "tile orientation must follow the operand storage");
  extern __shared__ double dsm[];
  // symmetric rank-k updates only need the tiles that touch the upper triangle
  if (upper_only && (int)(blockIdx.x + 1) * Cfg::BN <= (int)blockIdx.y * Cfg::BM) return;
  const int bz = blockIdx.z;
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  if (amap) amap += bz * sAm;
  if (bmap) bmap += bz * sBm;
  if (cmap) cmap += bz * sCm;
  const int m0 = blockIdx.y * Cfg::BM, n0 = blockIdx.x * Cfg::BN;
  struct AP {
    const double* A; int64_t lda; const int32_t* amap; int M, K, m0; bool vec;
    __device__ __forceinline__ void stage(double* As, int ks) {
      const int k0 = ks * Cfg::BK;
      if (TA) {
        if (amap) tile_copy<Cfg::NT>(As, Cfg::SA, A, lda, Cfg::BK, Cfg::BM, k0, m0, K, M, MappedRows{amap}, vec, 1);
        else tile_copy<Cfg::NT>(As, Cfg::SA, A, lda, Cfg::BK, Cfg::BM, k0, m0, K, M, IdentityRows{}, vec, 1);
      } else {
        if (amap) tile_copy<Cfg::NT>(As, Cfg::SA, A, lda, Cfg::BM, Cfg::BK, m0, k0, M, K, MappedRows{amap}, vec, 2);
        else tile_copy<Cfg::NT>(As, Cfg::SA, A, lda, Cfg::BM, Cfg::BK, m0, k0, M, K, IdentityRows{}, vec, 2);
      }
    }
  } ap{A, lda, amap, M, K, m0, vecA != 0};
  struct BP {
    const double* B; int64_t ldb; const int32_t* bmap; int N, K, n0; bool vec;
    __device__ __forceinline__ void stage(double* Bs, int ks) {
      const int k0 = ks * Cfg::BK;
      if (!TB) {
        if (bmap) tile_copy<Cfg::NT>(Bs, Cfg::SB, B, ldb, Cfg::BK, Cfg::BN, k0, n0, K, N, MappedRows{bmap}, vec, 1);
        else tile_copy<Cfg::NT>(Bs, Cfg::SB, B, ldb, Cfg::BK, Cfg::BN, k0, n0, K, N, IdentityRows{}, vec, 1);
      } else {
        if (bmap) tile_copy<Cfg::NT>(Bs, Cfg::SB, B, ldb, Cfg::BN, Cfg::BK, n0, k0, N, K, MappedRows{bmap}, vec, 2);
        else tile_copy<Cfg::NT>(Bs, Cfg::SB, B, ldb, Cfg::BN, Cfg::BK, n0, k0, N, K, IdentityRows{}, vec, 2);
      }
    }
  } bp{B, ldb, bmap, N, K, n0, vecB != 0};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
  // alpha = +-1 with beta != 0 (the trailing updates C -= A B): start the
  // accumulators from alpha*beta*C, loaded before the main loop so the C read
  // overlaps the operand prologue; the epilogue is then store-only.
  const bool preload = beta != 0.0 && (alpha == 1.0 || alpha == -1.0);
  const double ab = alpha * beta;
  // 16-byte C accesses when every fragment pair is aligned
  const bool cvec = ((((uintptr_t)C) | ((uintptr_t)(ldc * 8))) & 15) == 0;
  double acc[Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int r = m0 + wr * Cfg::WM + i * 8 + g;
    const double* crow = C + (int64_t)(r < M ? (cmap ? cmap[r] : r) : 0) * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      int c = n0 + wc * Cfg::WN + j * 8 + 2 * t;
      if (preload && r < M) {
        if (cvec && c + 1 < N) {
          double2 v = *reinterpret_cast<const double2*>(crow + c);
          acc[i][j][0] = ab * v.x;
          acc[i][j][1] = ab * v.y;
        } else {
          if (c < N) acc[i][j][0] = ab * crow[c];
          if (c + 1 < N) acc[i][j][1] = ab * crow[c + 1];
        }
      }
    }
  }
  WholeStage<decltype(ap)> apw{ap};
  dmma_mainloop<Cfg>(apw, bp, (K + Cfg::BK - 1) / Cfg::BK, dsm, acc);
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int r = m0 + wr * Cfg::WM + i * 8 + g;
    if (r >= M) continue;
    double* crow = C + (int64_t)(cmap ? cmap[r] : r) * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      int c = n0 + wc * Cfg::WN + j * 8 + 2 * t;
      if (preload) {
        if (cvec && c + 1 < N) {
          *reinterpret_cast<double2*>(crow + c) = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        } else {
          if (c < N) crow[c] = alpha * acc[i][j][0];
          if (c + 1 < N) crow[c + 1] = alpha * acc[i][j][1];
        }
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h >= N) continue;
        double v = alpha * acc[i][j][h];
        crow[c + h] = (beta == 0.0) ? v : fma(beta, crow[c + h], v);
      }
    }
  }
}

// tile_copy for a producer group: thread pt of NP copies a (rows x cols)
// tile, row r of the source is map[r] (or r), zero fill outside (rlim, clim).
// `free_dim` names the tile dimension that is NOT the product's k dimension
// (1: the contiguous one, 2: the row one): entries beyond its limit only
// reach outputs that are never stored, so they are left as they are instead
// of being zero-filled -- the zero-fill costs two 8-byte cp.async per
// 16-byte chunk, and the CTAs of a ragged last tile ran ~2x longer than the
// others (N = 4708: 31.8 TF/s against 34.2 for N = 4736 on the same grid).
template <int NP>
__device__ __forceinline__ void producer_copy(int pt, double* dst, int sstride, const double* src, int64_t ld,
                                              int rows, int cols, int r0, int c0, int rlim, int clim,
                                              const int32_t* map, bool vec2, int free_dim = 0) {
  if (vec2) {
    const int half = cols >> 1;
    for (int e = pt; e < rows * half; e += NP) {
      const int r = e / half, c = (e - r * half) * 2;
      const int gr = r0 + r, gc = c0 + c;
      double* d = dst + r * sstride + c;
      if (free_dim == 2 && gr >= rlim) continue;
      if (free_dim == 1 && gc >= clim) continue;
      const int64_t row = gr < rlim ? (int64_t)(map ? map[gr] : gr) : 0;
      if (gr < rlim && gc + 1 < clim) {
        cp_async16(d, src + row * ld + gc, true);
      } else {
        const bool ok = gr < rlim && gc < clim;
        cp_async8(d, ok ? (const void*)(src + row * ld + gc) : (const void*)src, ok);
        if (free_dim != 1 || gr >= rlim) cp_async8(d + 1, src, false);   // a k row past the end is zero in both halves
      }
    }
  } else {
    for (int e = pt; e < rows * cols; e += NP) {
      const int r = e / cols, c = e - r * cols;
      const int gr = r0 + r, gc = c0 + c;
      if (free_dim == 2 && gr >= rlim) continue;
      if (free_dim == 1 && gc >= clim) continue;
      const bool ok = gr < rlim && gc < clim;
      const int64_t row = ok ? (int64_t)(map ? map[gr] : gr) : 0;
      cp_async8(dst + r * sstride + c, ok ? (const void*)(src + row * ld + gc) : (const void*)src, ok);
    }
  }
}

// Warp-specialised batched GEMM (the k_apply3 structure with a stored A):
// NPROD producer threads move both operand tiles of a stage with cp.async
// (row maps, either orientation) and signal full[s] through
// cp.async.mbarrier.arrive; the consumer warps run the DMMAs from a
// STAGES-deep ring and release empty[s]. Producer address arithmetic and
// copy latency leave the consumers' issue slots (k_gemm2 interleaves both in
// every warp and waits on __syncthreads each step).
template <class Cfg, bool TA, bool TB, int NPROD>
__global__ void __launch_bounds__(Cfg::NT + NPROD, 1) k_gemm3(int M, int N, int K, double alpha,
                                                              const double* __restrict__ A, int64_t lda, int64_t sA,
                                                              const int32_t* __restrict__ amap, int64_t sAm,
                                                              const double* __restrict__ B, int64_t ldb, int64_t sB,
                                                              const int32_t* __restrict__ bmap, int64_t sBm,
                                                              double beta, double* __restrict__ C, int64_t ldc,
                                                              int64_t sC, const int32_t* __restrict__ cmap,
                                                              int64_t sCm, int vecA, int vecB, int upper_only) {
  static_assert(Cfg::A_KM == TA && Cfg::B_KM == !TB, "tile orientation must follow the operand storage");
  constexpr int STAGES = Cfg::STAGES, BK = Cfg::BK, NCONS = Cfg::NT;
  extern __shared__ double dsm[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  // CTAs are dispatched in launch order (x fastest), so a wave of 148 CTAs on
  // the natural (column tile, row tile) grid is a 148 / nx x nx slab that
  // streams nx column tiles of B for a few row tiles of A. Column tiles are
  // taken in groups of RASTER_GW instead, rows fastest inside a group: a wave
  // is then a ~12 x 12 block of tiles and reads 24 operand strips from DRAM
  // instead of nx + 148 / nx (the c3 strip GEMM, nx = 37: 41).
  constexpr int RASTER_GW = 12;
  int tile_n = blockIdx.x, tile_m = blockIdx.y;
  if ((int)gridDim.x > RASTER_GW && (int)gridDim.y > 1) {
    const int nx = gridDim.x, ny = gridDim.y;
    const int lin = blockIdx.y * nx + blockIdx.x;
    const int grp = lin / (RASTER_GW * ny), rem = lin - grp * (RASTER_GW * ny);
    const int gw = min(RASTER_GW, nx - grp * RASTER_GW);
    tile_m = rem / gw;
    tile_n = grp * RASTER_GW + rem - tile_m * gw;
  }
  if (upper_only && (tile_n + 1) * Cfg::BN <= tile_m * Cfg::BM) return;
  const int bz = blockIdx.z;
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  if (amap) amap += bz * sAm;
  if (bmap) bmap += bz * sBm;
  if (cmap) cmap += bz * sCm;
  const int m0 = tile_m * Cfg::BM, n0 = tile_n * Cfg::BN;
  const int nk = (K + BK - 1) / BK;
  double* As0 = dsm;
  double* Bs0 = dsm + STAGES * Cfg::A_STAGE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ws::mbar_init(&full[s], NPROD);
      ws::mbar_init(&empty[s], NCONS);
    }
  }
  __syncthreads();
  if ((int)threadIdx.x >= NCONS) {
    // ---------------- producers (threadIdx - NCONS in [0, NPROD))
    const int pt = threadIdx.x - NCONS;
    for (int ks = 0; ks < nk; ++ks) {
      const int s = ks % STAGES;
      ws::mbar_wait(&empty[s], ((uint32_t)(ks / STAGES) & 1) ^ 1);
      double* As = As0 + s * Cfg::A_STAGE;
      double* Bs = Bs0 + s * Cfg::B_STAGE;
      const int k0 = ks * BK;
      if (TA) producer_copy<NPROD>(pt, As, Cfg::SA, A, lda, BK, Cfg::BM, k0, m0, K, M, amap, vecA != 0, 1);
      else producer_copy<NPROD>(pt, As, Cfg::SA, A, lda, Cfg::BM, BK, m0, k0, M, K, amap, vecA != 0, 2);
      if (!TB) producer_copy<NPROD>(pt, Bs, Cfg::SB, B, ldb, BK, Cfg::BN, k0, n0, K, N, bmap, vecB != 0, 1);
      else producer_copy<NPROD>(pt, Bs, Cfg::SB, B, ldb, Cfg::BN, BK, n0, k0, N, K, bmap, vecB != 0, 2);
      ws::mbar_cp_async_arrive(&full[s]);
    }
    cp_async_wait<0>();
    return;
  }
  // ---------------- consumers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
  const int am0 = wr * Cfg::WM + g, bn0 = wc * Cfg::WN + g;
  const bool preload = beta != 0.0 && (alpha == 1.0 || alpha == -1.0);
  const double ab = alpha * beta;
  const bool cvec = ((((uintptr_t)C) | ((uintptr_t)(ldc * 8))) & 15) == 0;
  double acc[Cfg::MI][Cfg::NJ][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int r = m0 + wr * Cfg::WM + i * 8 + g;
    const double* crow = C + (int64_t)(r < M ? (cmap ? cmap[r] : r) : 0) * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      int c = n0 + wc * Cfg::WN + j * 8 + 2 * t;
      if (preload && r < M) {
        if (cvec && c + 1 < N) {
          double2 v = *reinterpret_cast<const double2*>(crow + c);
          acc[i][j][0] = ab * v.x;
          acc[i][j][1] = ab * v.y;
        } else {
          if (c < N) acc[i][j][0] = ab * crow[c];
          if (c + 1 < N) acc[i][j][1] = ab * crow[c + 1];
        }
      }
    }
  }
  for (int ks = 0; ks < nk; ++ks) {
    const int s = ks % STAGES;
    ws::mbar_wait(&full[s], (uint32_t)(ks / STAGES) & 1);
    const double* As = As0 + s * Cfg::A_STAGE;
    const double* Bs = Bs0 + s * Cfg::B_STAGE;
    double a[2][Cfg::MI], b[2][Cfg::NJ];
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i) a[0][i] = As[Cfg::ai(am0 + i * 8, t)];
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) b[0][j] = Bs[Cfg::bi(t, bn0 + j * 8)];
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int cur = k4 & 1;
      if (k4 + 1 < BK / 4) {
        const int kr = (k4 + 1) * 4 + t;
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i) a[cur ^ 1][i] = As[Cfg::ai(am0 + i * 8, kr)];
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) b[cur ^ 1][j] = Bs[Cfg::bi(kr, bn0 + j * 8)];
      }
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
    }
    ws::mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int r = m0 + wr * Cfg::WM + i * 8 + g;
    if (r >= M) continue;
    double* crow = C + (int64_t)(cmap ? cmap[r] : r) * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) {
      int c = n0 + wc * Cfg::WN + j * 8 + 2 * t;
      if (preload) {
        if (cvec && c + 1 < N) {
          *reinterpret_cast<double2*>(crow + c) = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        } else {
          if (c < N) crow[c] = alpha * acc[i][j][0];
          if (c + 1 < N) crow[c + 1] = alpha * acc[i][j][1];
        }
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h >= N) continue;
        double v = alpha * acc[i][j][h];
        crow[c + h] = (beta == 0.0) ? v : fma(beta, crow[c + h], v);
      }
    }
  }
}

template <int BM, int BN, int WMW, int WNW, int STAGES, int BK, int NPROD>
int launch_gemm3(int ta, int tb, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA,
                 const int32_t* amap, int64_t sAm, const double* B, int64_t ldb, int64_t sB, const int32_t* bmap,
                 int64_t sBm, double beta, double* C, int64_t ldc, int64_t sC, const int32_t* cmap, int64_t sCm,
                 int batch, cudaStream_t st, int upper_only = 0) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  auto aligned = [](const void* p, int64_t ld, int64_t stride) {
    return (((uintptr_t)p) % 16 == 0) && (ld % 2 == 0) && (stride % 2 == 0);
  };
  int vecA = aligned(A, lda, sA) ? 1 : 0;
  int vecB = aligned(B, ldb, sB) ? 1 : 0;
#define UBLR_G3(TA, TB)                                                                                       \
  {                                                                                                           \
    using Cfg = TileCfg<BM, BN, BK, WMW, WNW, STAGES, TA, !TB>;                                               \
    size_t sm = Cfg::smem_bytes();                                                                            \
    UBLR_CUDA(cudaFuncSetAttribute(k_gemm3<Cfg, TA, TB, NPROD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_gemm3<Cfg, TA, TB, NPROD><<<grid, Cfg::NT + NPROD, sm, st>>>(M, N, K, alpha, A, lda, sA, amap, sAm, B, ldb, sB, \
                                                                  bmap, sBm, beta, C, ldc, sC, cmap, sCm, vecA, vecB, \
                                                                  upper_only);                                 \
  }
  if (!ta && !tb) UBLR_G3(false, false)
  else if (!ta && tb) UBLR_G3(false, true)
  else if (ta && !tb) UBLR_G3(true, false)
  else UBLR_G3(true, true)
#undef UBLR_G3
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

template <int BM, int BN, int WMW, int WNW, int STAGES, int BK = 32, bool K8 = false>
int launch_gemm2(int ta, int tb, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA,
                 const int32_t* amap, int64_t sAm, const double* B, int64_t ldb, int64_t sB, const int32_t* bmap,
                 int64_t sBm, double beta, double* C, int64_t ldc, int64_t sC, const int32_t* cmap, int64_t sCm,
                 int batch, cudaStream_t st, int upper_only = 0) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  auto aligned = [](const void* p, int64_t ld, int64_t stride) {
    return (((uintptr_t)p) % 16 == 0) && (ld % 2 == 0) && (stride % 2 == 0);
  };
  int vecA = aligned(A, lda, sA) ? 1 : 0;
  int vecB = aligned(B, ldb, sB) ? 1 : 0;
#define UBLR_G2(TA, TB)                                                                                       \
  {                                                                                                           \
    using Cfg = TileCfg<BM, BN, BK, WMW, WNW, STAGES, TA, !TB, K8>;                                           \
    size_t sm = Cfg::smem_bytes();                                                                            \
    UBLR_CUDA(cudaFuncSetAttribute(k_gemm2<Cfg, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_gemm2<Cfg, TA, TB><<<grid, Cfg::NT, sm, st>>>(M, N, K, alpha, A, lda, sA, amap, sAm, B, ldb, sB, bmap, sBm,  \
                                                    beta, C, ldc, sC, cmap, sCm, vecA, vecB, upper_only);     \
  }
  if (!ta && !tb) UBLR_G2(false, false)
  else if (!ta && tb) UBLR_G2(false, true)
  else if (ta && !tb) UBLR_G2(true, false)
  else UBLR_G2(true, true)
#undef UBLR_G2
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

// ------------------------------------------------------------ small blocks
constexpr int FT = 256;

// in-place inverse of an upper-triangular nb x nb matrix in shared memory
// (column-oriented back substitution; X = U^-1 written to `inv` with ld nb)
__device__ void tri_inv_upper(const double* U, int ldu, double* inv, int nb) {
  // solve U X = I column by column; thread c owns column c
  for (int c = threadIdx.x; c < nb; c += blockDim.x) {
    for (int r = nb - 1; r >= 0; --r) {
      double s = (r == c) ? 1.0 : 0.0;
      for (int q = r + 1; q <= c; ++q) s -= U[r * ldu + q] * inv[q * nb + c];
      inv[r * nb + c] = (r <= c) ? s / U[r * ldu + r] : 0.0;
    }
  }
}

// unit lower-triangular inverse
__device__ void tri_inv_unit_lower(const double* L, int ldl, double* inv, int nb) {
  for (int c = threadIdx.x; c < nb; c += blockDim.x) {
    for (int r = 0; r < nb; ++r) {
      double s = (r == c) ? 1.0 : 0.0;
      for (int q = c; q < r; ++q) s -= L[r * ldl + q] * inv[q * nb + c];
      inv[r * nb + c] = (r >= c) ? s : 0.0;
    }
  }
}

__global__ void __launch_bounds__(FT) k_potrf_diag(double* A, int64_t lda, int64_t sA, int j0, int nb,
                                                   double* R, int64_t ldr, int64_t sR, double* Rinv,
                                                   int* status) {
  extern __shared__ double sm[];
  double* S = sm;               // nb x (nb+1)
  double* I = sm + nb * (nb + 1);
  const int ld = nb + 1;
  const int bz = blockIdx.x;
  double* Ab = A + bz * sA + (int64_t)j0 * lda + j0;
  for (int e = threadIdx.x; e < nb * nb; e += FT) S[(e / nb) * ld + e % nb] = Ab[(int64_t)(e / nb) * lda + e % nb];
  __syncthreads();
  // upper Cholesky, row-oriented right-looking: S = R^T R
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {
      double d = S[j * ld + j];
      if (!(d > 0.0)) { atomicExch(status, 1); d = 1.0; }
      S[j * ld + j] = sqrt(d);
    }
    __syncthreads();
    double piv = S[j * ld + j];
    for (int c = j + 1 + threadIdx.x; c < nb; c += FT) S[j * ld + c] /= piv;
    __syncthreads();
    for (int e = threadIdx.x; e < (nb - j - 1) * (nb - j - 1); e += FT) {
      int r = j + 1 + e / (nb - j - 1), c = j + 1 + e % (nb - j - 1);
      if (c >= r) S[r * ld + c] -= S[j * ld + r] * S[j * ld + c];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += FT) {
    int r = e / nb, c = e % nb;
    if (r > c) S[r * ld + c] = 0.0;
  }
  __syncthreads();
  tri_inv_upper(S, ld, I, nb);
  __syncthreads();
  double* Rb = R + bz * sR + (int64_t)j0 * ldr + j0;
  double* Ib = Rinv + (int64_t)bz * nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += FT) {
    int r = e / nb, c = e % nb;
    Rb[(int64_t)r * ldr + c] = S[r * ld + c];
    Ib[e] = I[e];
  }
}

__global__ void __launch_bounds__(FT) k_lu_sign_diag(double* W, int64_t ldw, int64_t sW, int j0, int nb,
                                                     double* LU, int64_t ldlu, int64_t sLU, double* Linv,
                                                     double* Uinv, double* D, int64_t sD, int* status,
                                                     const double* __restrict__ R, int64_t ldr, int64_t sR, int n) {
  extern __shared__ double sm[];
  double* S = sm;
  double* I = sm + nb * (nb + 1);
  const int ld = nb + 1;
  const int bz = blockIdx.x;
  double* Wb = W + bz * sW + (int64_t)j0 * ldw + j0;
  for (int e = threadIdx.x; e < nb * nb; e += FT) S[(e / nb) * ld + e % nb] = Wb[(int64_t)(e / nb) * ldw + e % nb];
  __syncthreads();
  const double* Rb = R ? R + bz * sR + (int64_t)j0 * ldr + j0 : nullptr;
  __shared__ double dsh;
  for (int j = 0; j < nb; ++j) {
    if (!Rb) {
      if (threadIdx.x == 0) {
        // working matrix W = -Q (eliminated so far); D_jj = -sign(q_jj) = sign(w_jj)
        // makes the pivot w + D_jj of magnitude |w| + 1
        double w = S[j * ld + j];
        double d = (w > 0.0) ? 1.0 : -1.0;
        S[j * ld + j] = w + d;
        D[bz * sD + j0 + j] = d;
      }
    } else {
      // R-scaled form: the matrix is D R - B1^T = (D - Q_top) R; row j of D R
      // enters when j becomes the pivot row (earlier multipliers never read it,
      // R being upper triangular). Same sign rule: sign(w'_jj) = sign(w_jj).
      if (threadIdx.x == 0) {
        double w = S[j * ld + j];
        double d = (w > 0.0) ? 1.0 : -1.0;
        dsh = d;
        D[bz * sD + j0 + j] = d;
      }
      __syncthreads();
      const double d = dsh;
      for (int c = j + threadIdx.x; c < nb; c += FT) S[j * ld + c] = fma(d, Rb[(int64_t)j * ldr + c], S[j * ld + c]);
    }
    __syncthreads();
    double piv = S[j * ld + j];
    if (piv == 0.0) atomicExch(status, 1);
    for (int r = j + 1 + threadIdx.x; r < nb; r += FT) S[r * ld + j] /= piv;
    __syncthreads();
    for (int e = threadIdx.x; e < (nb - j - 1) * (nb - j - 1); e += FT) {
      int r = j + 1 + e / (nb - j - 1), c = j + 1 + e % (nb - j - 1);
      S[r * ld + c] -= S[r * ld + j] * S[j * ld + c];
    }
    __syncthreads();
  }
  double* LUb = LU + bz * sLU + (int64_t)j0 * ldlu + j0;
  for (int e = threadIdx.x; e < nb * nb; e += FT) LUb[(int64_t)(e / nb) * ldlu + e % nb] = S[(e / nb) * ld + e % nb];
  if (Rb) {
    // the panel rows' D R to the right of the block, before U12 = L11^-1 W12
    const int rest = n - j0 - nb;
    double* Wb2 = Wb + nb;
    const double* Rb2 = Rb + nb;
    for (int r = 0; r < nb; ++r) {
      const double d = D[bz * sD + j0 + r];
      for (int c = threadIdx.x; c < rest; c += FT)
        Wb2[(int64_t)r * ldw + c] = fma(d, Rb2[(int64_t)r * ldr + c], Wb2[(int64_t)r * ldw + c]);
    }
  }
  tri_inv_unit_lower(S, ld, I, nb);
  __syncthreads();
  double* Lb = Linv + (int64_t)bz * nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += FT) Lb[e] = I[e];
  __syncthreads();
  tri_inv_upper(S, ld, I, nb);
  __syncthreads();
  double* Ub = Uinv + (int64_t)bz * nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += FT) Ub[e] = I[e];
}

// ------------------------------------------------- register-tile leaves
// 64 x 64 diagonal-block factorisations for nb <= 64 with the block held in
// registers: 256 threads in a 16 x 16 grid, thread (tr, tc) owns rows
// 4 tr .. 4 tr + 3 and columns 4 tc .. 4 tc + 3. Step j broadcasts the pivot
// row (and column) through a double-buffered shared-memory vector, so each
// elimination step costs one barrier; the 16 threads of a row group are one
// half-warp and read the pivot by shuffle. Rows / columns past nb are padded
// with the identity and never stored. The triangular inverses are
// Gauss-Jordan sweeps in the same layout. (The shared-memory kernels above,
// one barrier-separated phase per step with an integer division per entry
// and a thread per column in the inverses, stay for 64 < nb <= 96.)
struct RegTile {
  int tr, tc;
  __device__ __forceinline__ RegTile() : tr(threadIdx.x >> 4), tc(threadIdx.x & 15) {}
  __device__ __forceinline__ unsigned half_mask() const { return (tr & 1) ? 0xffff0000u : 0x0000ffffu; }
  // lane of thread (row group tr, column group c) inside this thread's warp
  __device__ __forceinline__ int lane_of(int c) const { return ((tr & 1) << 4) + c; }
};

// backward Gauss-Jordan: x <- U^-1 (x starts as the identity), U upper
// triangular held in u (only the upper part is read); rinv[a] = 1 / U[r][r]
// for the thread's rows r = 4 tr + a (kept from the factorisation: the
// serial chain of each step carries no division)
__device__ __forceinline__ void regtile_inv_upper(const RegTile& T, const double (&u)[4][4], const double (&rinv)[4],
                                                  double (&x)[4][4], double (*rowb)[64], double (*colb)[64]) {
  for (int jb = 15; jb >= 0; --jb) {
#pragma unroll
    for (int jj = 3; jj >= 0; --jj) {
      const int j = 4 * jb + jj, buf = j & 1;
      if (T.tr == jb) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          x[jj][b] = x[jj][b] * rinv[jj];
          rowb[buf][4 * T.tc + b] = x[jj][b];
        }
      }
      if (T.tc == jb) {
#pragma unroll
        for (int a = 0; a < 4; ++a) colb[buf][4 * T.tr + a] = u[a][jj];
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (4 * T.tr + a >= j) continue;
        const double m = colb[buf][4 * T.tr + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) x[a][b] = fma(-m, rowb[buf][4 * T.tc + b], x[a][b]);
      }
    }
  }
}

// forward Gauss-Jordan: x <- L^-1 (x starts as the identity), L unit lower
// triangular held in the strictly lower part of l
__device__ __forceinline__ void regtile_inv_unit_lower(const RegTile& T, const double (&l)[4][4], double (&x)[4][4],
                                                       double (*rowb)[64], double (*colb)[64]) {
  for (int jb = 0; jb < 16; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj, buf = j & 1;
      if (T.tr == jb) {
#pragma unroll
        for (int b = 0; b < 4; ++b) rowb[buf][4 * T.tc + b] = x[jj][b];
      }
      if (T.tc == jb) {
#pragma unroll
        for (int a = 0; a < 4; ++a) colb[buf][4 * T.tr + a] = l[a][jj];
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (4 * T.tr + a <= j) continue;
        const double m = colb[buf][4 * T.tr + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) x[a][b] = fma(-m, rowb[buf][4 * T.tc + b], x[a][b]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_potrf64(double* A, int64_t lda, int64_t sA, int j0, int nb, double* R,
                                                 int64_t ldr, int64_t sR, double* Rinv, int* status) {
  __shared__ double rowb[2][64], colb[2][64];
  const RegTile T;
  const int bz = blockIdx.x;
  const double* Ab = A + bz * sA + (int64_t)j0 * lda + j0;
  double v[4][4], x[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      v[a][b] = (r < nb && c < nb) ? Ab[(int64_t)r * lda + c] : (r == c ? 1.0 : 0.0);
      x[a][b] = r == c ? 1.0 : 0.0;
    }
  bool bad = false;
  double rinv[4] = {1.0, 1.0, 1.0, 1.0};   // 1 / R[r][r] of this thread's rows
  // upper Cholesky, right-looking by rows: R[j, j:] = S[j, j:] / sqrt(S[j, j]),
  // S[r, c] -= R[j, r] R[j, c] for j < r <= c
  for (int jb = 0; jb < 16; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj, buf = j & 1;
      if (T.tr == jb) {
        double s2 = __shfl_sync(T.half_mask(), v[jj][jj], T.lane_of(jb));
        if (!(s2 > 0.0)) {
          bad = true;
          s2 = 1.0;
        }
        const double rs = rsqrt(s2);          // 1 / R[j][j]
        const double d = s2 * rs;             // R[j][j]
        rinv[jj] = rs;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = 4 * T.tc + b;
          v[jj][b] = c > j ? v[jj][b] * rs : (c == j ? d : 0.0);
          rowb[buf][c] = v[jj][b];
        }
      }
      __syncthreads();
      double rc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) rc[b] = rowb[buf][4 * T.tc + b];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = 4 * T.tr + a;
        if (r <= j) continue;
        const double rr = rowb[buf][r];
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * T.tc + b >= r) v[a][b] = fma(-rr, rc[b], v[a][b]);
      }
    }
  }
  if (bad) atomicExch(status, 1);
  __syncthreads();   // the last step's broadcast vectors are read before the inverse reuses them
  regtile_inv_upper(T, v, rinv, x, rowb, colb);
  double* Rb = R + bz * sR + (int64_t)j0 * ldr + j0;
  double* Ib = Rinv + (int64_t)bz * nb * nb;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      if (r < nb && c < nb) {
        Rb[(int64_t)r * ldr + c] = r > c ? 0.0 : v[a][b];
        Ib[r * nb + c] = x[a][b];
      }
    }
}

__global__ void __launch_bounds__(256) k_lu_sign64(double* W, int64_t ldw, int64_t sW, int j0, int nb, double* LU,
                                                   int64_t ldlu, int64_t sLU, double* Linv, double* Uinv, double* D,
                                                   int64_t sD, int* status, const double* __restrict__ R, int64_t ldr,
                                                   int64_t sR, int n) {
  __shared__ double rowb[2][64], colb[2][64];
  const RegTile T;
  const int bz = blockIdx.x;
  double* Wb = W + bz * sW + (int64_t)j0 * ldw + j0;
  const double* Rb = R ? R + bz * sR + (int64_t)j0 * ldr + j0 : nullptr;
  double v[4][4], rt[4][4];   // W tile; R tile (row j of D R joins at step j: loaded up front)
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      v[a][b] = (r < nb && c < nb) ? Wb[(int64_t)r * ldw + c] : (r == c ? 1.0 : 0.0);
      rt[a][b] = Rb ? ((r < nb && c < nb) ? Rb[(int64_t)r * ldr + c] : (r == c ? 1.0 : 0.0)) : 0.0;
    }
  bool bad = false;
  __shared__ double rpivb[2];
  double rinv[4] = {1.0, 1.0, 1.0, 1.0};   // 1 / U[r][r] of this thread's rows
  for (int jb = 0; jb < 16; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj, buf = j & 1;
      if (T.tr == jb) {
        // D_jj = sign(w_jj) (the working matrix is -Q eliminated so far);
        // plain form: pivot w + D_jj; R-scaled form: row j of D R joins now
        const double w = __shfl_sync(T.half_mask(), v[jj][jj], T.lane_of(jb));
        const double d = (w > 0.0) ? 1.0 : -1.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = 4 * T.tc + b;
          if (Rb) {
            if (c >= j) v[jj][b] = fma(d, rt[jj][b], v[jj][b]);
          } else if (c == j) {
            v[jj][b] = w + d;
          }
          rowb[buf][c] = v[jj][b];
        }
        // the pivot's reciprocal, from its owner (correctly rounded)
        const double pv = __shfl_sync(T.half_mask(), v[jj][jj], T.lane_of(jb));
        rinv[jj] = __drcp_rn(pv);
        if (T.tc == jb) {
          rpivb[buf] = rinv[jj];
          if (j < nb) D[bz * sD + j0 + j] = d;
        }
      }
      if (T.tc == jb) {
#pragma unroll
        for (int a = 0; a < 4; ++a) colb[buf][4 * T.tr + a] = v[a][jj];
      }
      __syncthreads();
      if (rowb[buf][j] == 0.0) bad = true;
      const double rpiv = rpivb[buf];
      double rc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) rc[b] = rowb[buf][4 * T.tc + b];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = 4 * T.tr + a;
        if (r <= j) continue;
        const double m = colb[buf][r] * rpiv;
        if (T.tc == jb) v[a][jj] = m;                 // L multiplier, stored in place
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * T.tc + b > j) v[a][b] = fma(-m, rc[b], v[a][b]);
      }
    }
  }
  if (bad && T.tr == 0 && T.tc == 0) atomicExch(status, 1);
  double* LUb = LU + bz * sLU + (int64_t)j0 * ldlu + j0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      if (r < nb && c < nb) LUb[(int64_t)r * ldlu + c] = v[a][b];
    }
  if (Rb && n > j0 + nb) {
    // the panel rows' D R to the right of the block, before U12 = L11^-1 W12
    __syncthreads();   // D of the panel written
    const int rest = n - j0 - nb;
    for (int r = 0; r < nb; ++r) {
      const double d = D[bz * sD + j0 + r];
      for (int c = threadIdx.x; c < rest; c += blockDim.x)
        Wb[(int64_t)r * ldw + nb + c] = fma(d, Rb[(int64_t)r * ldr + nb + c], Wb[(int64_t)r * ldw + nb + c]);
    }
  }
  double x[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) x[a][b] = (4 * T.tr + a == 4 * T.tc + b) ? 1.0 : 0.0;
  __syncthreads();   // the last elimination step's broadcast vectors are read
  regtile_inv_unit_lower(T, v, x, rowb, colb);
  double* Lb = Linv + (int64_t)bz * nb * nb;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      if (r < nb && c < nb) Lb[r * nb + c] = x[a][b];
      x[a][b] = r == c ? 1.0 : 0.0;
    }
  __syncthreads();
  regtile_inv_upper(T, v, rinv, x, rowb, colb);
  double* Ub = Uinv + (int64_t)bz * nb * nb;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * T.tr + a, c = 4 * T.tc + b;
      if (r < nb && c < nb) Ub[r * nb + c] = x[a][b];
    }
}

// out[b][r][c] = src[b*s_src + map[b*s_map + r] * ld + col0 + c]   (transpose: out[b][c][r])
// 32 x 32 tiles per CTA (32 x 8 threads), 32-bit tile indices; the
// transpose goes through a padded shared-memory tile so that both the read
// (along c) and the write (along r) are coalesced.
__global__ void __launch_bounds__(256) k_gather(const double* __restrict__ src, int64_t ld, int64_t s_src,
                                                const int32_t* __restrict__ map, int64_t s_map, int rows, int cols,
                                                int col0, int transpose, double* __restrict__ out, int64_t ldo,
                                                int64_t s_out) {
  __shared__ double tile[32][33];
  const int bz = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const double* sb = src + bz * s_src + col0;
  const int32_t* mb = map ? map + bz * s_map : nullptr;
  double* ob = out + bz * s_out;
  if (!transpose) {
    const int c = c0 + tx;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + ty + 8 * i;
      if (r < rows && c < cols) {
        const int64_t pr = mb ? mb[r] : r;
        ob[(int64_t)r * ldo + c] = sb[pr * ld + c];
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i, c = c0 + tx;
    if (r < rows && c < cols) {
      const int64_t pr = mb ? mb[r] : r;
      tile[ty + 8 * i][tx] = sb[pr * ld + c];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, r = r0 + tx;
    if (r < rows && c < cols) ob[(int64_t)c * ldo + r] = tile[tx][ty + 8 * i];
  }
}

// W[b][r][c] += d[b*s_d + r] * R[b][r][c] on a rows x cols sub-block
__global__ void __launch_bounds__(256) k_add_scaled_rows(double* __restrict__ W, int64_t ldw, int64_t s_w,
                                                         const double* __restrict__ R, int64_t ldr, int64_t s_r,
                                                         const double* __restrict__ d, int64_t s_d, int rows,
                                                         int cols) {
  const int bz = blockIdx.z;
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    double* w = W + bz * s_w + (int64_t)r * ldw + c;
    *w = fma(d[bz * s_d + r], R[bz * s_r + (int64_t)r * ldr + c], *w);
  }
}

// X[b][r][c] *= d[b*s_d + r]
__global__ void __launch_bounds__(256) k_scale_rows(double* __restrict__ X, int64_t ldx, int64_t s_x,
                                                    const double* __restrict__ d, int64_t s_d, int rows, int cols) {
  const int bz = blockIdx.z;
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) X[bz * s_x + (int64_t)r * ldx + c] *= d[bz * s_d + r];
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int ublr_gather(const double* src, int64_t ld, int64_t s_src, const int32_t* map, int64_t s_map, int rows,
                           int cols, int col0, int transpose, double* out, int64_t ldo, int64_t s_out, int batch,
                           void* stream) {
  UBLR_REQUIRE(src && out && rows >= 0 && cols >= 0 && batch >= 0 && batch <= 65535, UBLR_ERR_VALUE,
               "ublr_gather: bad arguments");
  if (!rows || !cols || !batch) return UBLR_OK;
  UBLR_REQUIRE((rows + 31) / 32 <= 65535, UBLR_ERR_VALUE, "ublr_gather: too many rows");
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), batch);
  k_gather<<<grid, 256, 0, (cudaStream_t)stream>>>(src, ld, s_src, map, s_map, rows, cols, col0, transpose, out, ldo,
                                                   s_out);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_add_scaled_rows(double* W, int64_t ldw, int64_t s_w, const double* R, int64_t ldr, int64_t s_r,
                                    const double* d, int64_t s_d, int rows, int cols, int batch, void* stream) {
  UBLR_REQUIRE(W && R && d && rows >= 0 && cols >= 0 && batch >= 0 && batch <= 65535, UBLR_ERR_VALUE,
               "ublr_add_scaled_rows: bad arguments");
  if (!rows || !cols || !batch) return UBLR_OK;
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)(rows < 64 ? rows : 64), batch);
  k_add_scaled_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(W, ldw, s_w, R, ldr, s_r, d, s_d, rows, cols);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_scale_rows(double* X, int64_t ldx, int64_t s_x, const double* d, int64_t s_d, int rows, int cols,
                               int batch, void* stream) {
  UBLR_REQUIRE(X && d && rows >= 0 && cols >= 0 && batch >= 0 && batch <= 65535, UBLR_ERR_VALUE,
               "ublr_scale_rows: bad arguments");
  if (!rows || !cols || !batch) return UBLR_OK;
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)(rows < 256 ? rows : 256), batch);
  k_scale_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(X, ldx, s_x, d, s_d, rows, cols);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_gemm_batched(int ta, int tb, int M, int N, int K, double alpha, const double* A, int64_t lda,
                                 int64_t sA, const int32_t* amap, int64_t sAm, const double* B, int64_t ldb,
                                 int64_t sB, const int32_t* bmap, int64_t sBm, double beta, double* C, int64_t ldc,
                                 int64_t sC, const int32_t* cmap, int64_t sCm, int batch, void* stream) {
  UBLR_REQUIRE(M >= 0 && N >= 0 && K >= 0 && batch >= 0 && A && B && C, UBLR_ERR_VALUE, "ublr_gemm_batched: bad arguments");
  UBLR_REQUIRE(batch <= 65535, UBLR_ERR_VALUE, "ublr_gemm_batched: batch <= 65535");
  if (M == 0 || N == 0 || batch == 0) return UBLR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t tiles128 = (int64_t)((M + 127) / 128) * ((N + 127) / 128) * batch;
  // tile configuration. Default (6): the warp-specialised k_gemm3 for large
  // tiles (128 x 128, 8 consumer warps, 4 producer warps, 3 stages of BK 32:
  // 33.4 TF/s = 90 % of the DMMA peak on 4096^3 and the c3 Gram / Cholesky
  // shapes, against 27.5 TF/s for k_gemm2; tools/gemm_bench.py,
  // profiles/r02/gemm_bench.txt) and k_gemm2 64 x 64 for skinny / small
  // products, where the synchronous kernel is faster. UBLR_GEMM_CFG selects
  // alternatives for benchmarking: 0 k_gemm2 everywhere (BK 32, 2 stages);
  // 1 / 2 / 3 k_gemm2 with BK 16 x 4 stages / + m16n8k8 / BK 32 x 3 stages;
  // 4 / 5 k_gemm3 with BK 16 x 4 stages (8 / 16 consumer warps).
  static const int cfg = [] {
    const char* e = getenv("UBLR_GEMM_CFG");
    return e ? atoi(e) : 6;
  }();
#define UBLR_GEMM_ARGS ta, tb, M, N, K, alpha, A, lda, sA, amap, sAm, B, ldb, sB, bmap, sBm, beta, C, ldc, sC, cmap, sCm, batch, st
  if (M >= 96 && N >= 96 && tiles128 >= 148) {
    if (cfg == 1) return launch_gemm2<128, 128, 4, 4, 4, 16>(UBLR_GEMM_ARGS);
    if (cfg == 2) return launch_gemm2<128, 128, 4, 4, 4, 16, true>(UBLR_GEMM_ARGS);
    if (cfg == 3) return launch_gemm2<128, 128, 4, 4, 3, 32>(UBLR_GEMM_ARGS);
    if (cfg == 4) return launch_gemm3<128, 128, 4, 2, 4, 16, 128>(UBLR_GEMM_ARGS);
    if (cfg == 5) return launch_gemm3<128, 128, 4, 4, 4, 16, 128>(UBLR_GEMM_ARGS);
    if (cfg == 6) return launch_gemm3<128, 128, 4, 2, 3, 32, 128>(UBLR_GEMM_ARGS);
    return launch_gemm2<128, 128, 4, 4, 2>(UBLR_GEMM_ARGS);
  }
  // skinny products (N <= 48: the k-column null-space solves and sample
  // products of block nullification): 128 x 40 / 128 x 48 k_gemm2 tiles,
  // 8 warps of 16 x N, instead of the 64 x 64 tile whose last columns are
  // padding: 15.8 -> 26.5 TF/s on M 2354 x N 40 x K 2304 (batch 98), 18.1 ->
  // 28.3 on 2304 x 40 x 2304 (a 3-stage ring: 19.6 / 21.1; a 128 x 48
  // k_gemm3: 15.8). UBLR_GEMM_SKINNY=0 restores the 64 x 64 tile.
  static const int skinny = [] {
    const char* e = getenv("UBLR_GEMM_SKINNY");
    return e ? atoi(e) : 1;
  }();
  if (skinny && N <= 40 && M >= 128) return launch_gemm2<128, 40, 8, 1, 2>(UBLR_GEMM_ARGS);
  if (skinny && N <= 48 && M >= 128) return launch_gemm2<128, 48, 8, 1, 2>(UBLR_GEMM_ARGS);
  if (cfg == 1) return launch_gemm2<64, 64, 2, 4, 4, 16>(UBLR_GEMM_ARGS);
  if (cfg == 2) return launch_gemm2<64, 64, 2, 4, 4, 16, true>(UBLR_GEMM_ARGS);
  if (cfg == 3) return launch_gemm2<64, 64, 2, 4, 3, 32>(UBLR_GEMM_ARGS);
  if (cfg == 4 || cfg == 5) return launch_gemm3<64, 64, 2, 2, 4, 16, 64>(UBLR_GEMM_ARGS);
  return launch_gemm2<64, 64, 2, 4, 2>(UBLR_GEMM_ARGS);
#undef UBLR_GEMM_ARGS
}

extern "C" int ublr_syrk_upper_batched(int M, int K, double alpha, const double* A, int64_t lda, int64_t sA,
                                       double beta, double* C, int64_t ldc, int64_t sC, int batch, void* stream) {
  UBLR_REQUIRE(M >= 0 && K >= 0 && batch >= 0 && A && C, UBLR_ERR_VALUE, "ublr_syrk_upper_batched: bad arguments");
  UBLR_REQUIRE(batch <= 65535, UBLR_ERR_VALUE, "ublr_syrk_upper_batched: batch <= 65535");
  if (M == 0 || batch == 0) return UBLR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t tiles128 = (int64_t)((M + 127) / 128) * ((M + 127) / 128) * batch / 2;
  if (M >= 96 && tiles128 >= 148)
    return launch_gemm3<128, 128, 4, 2, 3, 32, 128>(1, 0, M, M, K, alpha, A, lda, sA, nullptr, 0, A, lda, sA, nullptr,
                                                    0, beta, C, ldc, sC, nullptr, 0, batch, st, 1);
  return launch_gemm2<64, 64, 2, 4, 2>(1, 0, M, M, K, alpha, A, lda, sA, nullptr, 0, A, lda, sA, nullptr, 0, beta, C,
                                       ldc, sC, nullptr, 0, batch, st, 1);
}

// leaf kernels: 2 = register-tile (nb <= 64, default), 1 = shared-memory
static int leaf_version() {
  static const int v = [] {
    const char* e = getenv("UBLR_LEAF_VERSION");
    return e ? atoi(e) : 2;
  }();
  return v;
}

extern "C" int ublr_potrf_diag(double* A, int64_t lda, int64_t sA, int j0, int nb, double* R, int64_t ldr,
                               int64_t sR, double* Rinv, int* status, int batch, void* stream) {
  UBLR_REQUIRE(A && R && Rinv && status && nb >= 1 && nb <= 96 && batch >= 1, UBLR_ERR_VALUE,
               "ublr_potrf_diag: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (nb <= 64 && leaf_version() == 2) {
    k_potrf64<<<batch, 256, 0, st>>>(A, lda, sA, j0, nb, R, ldr, sR, Rinv, status);
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
  size_t sm = (size_t)(nb * (nb + 1) + nb * nb) * sizeof(double);
  UBLR_CUDA(cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_potrf_diag<<<batch, FT, sm, st>>>(A, lda, sA, j0, nb, R, ldr, sR, Rinv, status);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

extern "C" int ublr_lu_sign_diag(double* W, int64_t ldw, int64_t sW, int j0, int nb, double* LU, int64_t ldlu,
                                 int64_t sLU, double* Linv, double* Uinv, double* D, int64_t sD, int* status,
                                 int batch, void* stream) {
  return ublr_lu_sign_diag_r(W, ldw, sW, j0, nb, LU, ldlu, sLU, Linv, Uinv, D, sD, status, nullptr, 0, 0, 0, batch,
                             stream);
}

extern "C" int ublr_lu_sign_diag_r(double* W, int64_t ldw, int64_t sW, int j0, int nb, double* LU, int64_t ldlu,
                                   int64_t sLU, double* Linv, double* Uinv, double* D, int64_t sD, int* status,
                                   const double* R, int64_t ldr, int64_t sR, int n, int batch, void* stream) {
  UBLR_REQUIRE(W && LU && Linv && Uinv && D && status && nb >= 1 && nb <= 96 && batch >= 1, UBLR_ERR_VALUE,
               "ublr_lu_sign_diag: bad arguments");
  UBLR_REQUIRE(!R || n >= j0 + nb, UBLR_ERR_VALUE, "ublr_lu_sign_diag_r: n < j0 + nb");
  cudaStream_t st = (cudaStream_t)stream;
  if (nb <= 64 && leaf_version() == 2) {
    k_lu_sign64<<<batch, 256, 0, st>>>(W, ldw, sW, j0, nb, LU, ldlu, sLU, Linv, Uinv, D, sD, status, R, ldr, sR, n);
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
  size_t sm = (size_t)(nb * (nb + 1) + nb * nb) * sizeof(double);
  UBLR_CUDA(cudaFuncSetAttribute(k_lu_sign_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_lu_sign_diag<<<batch, FT, sm, st>>>(W, ldw, sW, j0, nb, LU, ldlu, sLU, Linv, Uinv, D, sD, status, R, ldr, sR,
                                         n);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}

// ------------------------------------------------------------ Gram assembly
// G_c (n x n, n = nb * m) for chunk entry c from shared block products:
// block (a, b) of G_c is P[pid] (m x m) if pid = map[c][a][b] >= 0, or the
// transpose of P[-pid - 1] otherwise (Omega_j Omega_j'^T is computed once per
// neighbouring pair and reused by every neighbourhood containing both).
namespace ublr {
namespace {
__global__ void __launch_bounds__(256) k_assemble_gram(const double* __restrict__ P, const int32_t* __restrict__ map,
                                                       int nb, int m, double* __restrict__ G) {
  // CTA = one 32 x 32 tile of block (a, b) of G_c; transposed blocks go
  // through a shared-memory tile (coalesced read and write)
  __shared__ double tile[32][33];
  const int c = blockIdx.z;
  const int n = nb * m;
  const int tpb = (m + 31) / 32;                    // tiles per block side
  const int ab = blockIdx.y, a = ab / nb, b = ab - a * nb;
  const int ty0 = blockIdx.x / tpb, tx0 = blockIdx.x - ty0 * tpb;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int pid = map[((int64_t)c * nb + a) * nb + b];
  double* Gc = G + (int64_t)c * n * n + (int64_t)(a * m) * n + b * m;
  if (pid >= 0) {
    const double* Pb = P + (int64_t)pid * m * m;
    const int q = tx0 * 32 + tx;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty0 * 32 + ty + 8 * i;
      if (r < m && q < m) Gc[(int64_t)r * n + q] = Pb[(int64_t)r * m + q];
    }
    return;
  }
  const double* Pb = P + (int64_t)(-pid - 1) * m * m;   // G block (r, q) = P[q][r]
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = tx0 * 32 + ty + 8 * i, r = ty0 * 32 + tx;
    if (q < m && r < m) tile[ty + 8 * i][tx] = Pb[(int64_t)q * m + r];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty0 * 32 + ty + 8 * i, q = tx0 * 32 + tx;
    if (r < m && q < m) Gc[(int64_t)r * n + q] = tile[tx][ty + 8 * i];
  }
}
}  // namespace
}  // namespace ublr

extern "C" int ublr_assemble_gram(const double* P, const int32_t* map, int nb, int m, double* G, int batch,
                                  void* stream) {
  UBLR_REQUIRE(P && map && G && nb > 0 && m > 0 && batch > 0 && batch <= 65535, UBLR_ERR_VALUE,
               "ublr_assemble_gram: bad arguments");
  const int tpb = (m + 31) / 32;
  dim3 grid((unsigned)(tpb * tpb), (unsigned)(nb * nb), batch);
  k_assemble_gram<<<grid, 256, 0, (cudaStream_t)stream>>>(P, map, nb, m, G);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
