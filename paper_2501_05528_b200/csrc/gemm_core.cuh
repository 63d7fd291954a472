// Shared fp64 DMMA main loop for the operator-apply and batched GEMM kernels.
//
// CTA tile BM x BN, k-step BK, WMW x WNW warps, each warp owning a
// (BM/WMW) x (BN/WNW) tile of m8n8k4 accumulators. Each operand tile is kept
// in shared memory in the orientation its global source is contiguous in
// (so cp.async can move 16-byte chunks):
//   A k-major As[k][m] (stride BM+4)  or m-major As[m][k] (stride BK+4),
//   B k-major Bs[k][n] (stride BN+4)  or n-major Bs[n][k] (stride BK+4).
// With those +4 pads the fragment loads (lane (g, t) reads A[m0+g][k0+t],
// B[k0+t][n0+g]) are bank-conflict-free in both orientations.
// A STAGES-deep ring lets the producers (cp.async for stored operands,
// in-register generation for operator tiles) fill stage ks+STAGES-1 while
// the tensor pipe consumes stage ks; the fragments of the next k4 slice are
// loaded before the current slice's DMMAs issue.
#pragma once
#include "common.cuh"

#ifndef UBLR_MMA_K8
#define UBLR_MMA_K8 0
#endif

namespace ublr {

template <int BM_, int BN_, int BK_, int WMW_, int WNW_, int STAGES_, bool A_KM_ = true, bool B_KM_ = true,
          bool K8_ = false>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WMW = WMW_, WNW = WNW_, STAGES = STAGES_;
  static constexpr bool K8 = K8_;   // m16n8k8 DMMA instead of m8n8k4
  static constexpr bool A_KM = A_KM_, B_KM = B_KM_;
  static constexpr int NT = WMW * WNW * 32;
  static constexpr int SA = A_KM ? BM + 4 : BK + 4;  // row stride of the A tile in smem
  static constexpr int SB = B_KM ? BN + 4 : BK + 4;
  static constexpr int WM = BM / WMW;
  static constexpr int WN = BN / WNW;
  static constexpr int MI = WM / 8;
  static constexpr int NJ = WN / 8;
  static constexpr int A_STAGE = A_KM ? BK * SA : BM * SA;  // doubles
  static constexpr int B_STAGE = B_KM ? BK * SB : BN * SB;
  static constexpr size_t smem_bytes() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double); }
  // smem index of A(m, k) / B(k, n) inside one stage
  __device__ static __forceinline__ int ai(int m, int k) { return A_KM ? k * SA + m : m * SA + k; }
  __device__ static __forceinline__ int bi(int k, int n) { return B_KM ? k * SB + n : n * SB + k; }
};

// acc += A_tile * B_tile over nk k-steps. Producers fill one stage:
//   ap.stage(double* As, int ks);  bp.stage(double* Bs, int ks)
// (indexing through Cfg::ai / Cfg::bi) and may issue cp.async; one commit
// group per stage is made here.
template <class Cfg, class AP, class BP>
__device__ __forceinline__ void dmma_mainloop(AP& ap, BP& bp, int nk, double* smem,
                                              double (&acc)[Cfg::MI][Cfg::NJ][2]) {
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  double* As0 = smem;
  double* Bs0 = smem + STAGES * Cfg::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / Cfg::WNW, wc = warp % Cfg::WNW;
  const int am0 = wr * Cfg::WM + g;
  const int bn0 = wc * Cfg::WN + g;

  // producers may stage per-k-step side data (column coordinates) one step ahead
#pragma unroll
  for (int s = 0; s < STAGES; ++s)
    if (s < nk) ap.prefetch(s);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      ap.stage(As0 + s * Cfg::A_STAGE, s);
      bp.stage(Bs0 + s * Cfg::B_STAGE, s);
    }
    cp_async_commit();
  }
  for (int ks = 0; ks < nk; ++ks) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nx = ks + STAGES - 1;
    double* As_nx = As0 + (nx % STAGES) * Cfg::A_STAGE;
    if (nx < nk) bp.stage(Bs0 + (nx % STAGES) * Cfg::B_STAGE, nx);
    if (nx + 1 < nk) ap.prefetch(nx + 1);
    const double* As = As0 + (ks % STAGES) * Cfg::A_STAGE;
    const double* Bs = Bs0 + (ks % STAGES) * Cfg::B_STAGE;
    if constexpr ((UBLR_MMA_K8 || Cfg::K8) && Cfg::MI % 2 == 0) {
    // m16n8k8: 8-row groups (2i, 2i+1) of acc form one 16-row MMA tile
    constexpr int MI2 = Cfg::MI / 2;
    // single-buffered fragments (the double-buffered form spills at 128
    // registers); ptxas hoists the next slice's loads over these MMAs
#pragma unroll
    for (int k8 = 0; k8 < BK / 8; ++k8) {
      const int k0 = k8 * 8;
      double a[MI2][4], b[Cfg::NJ][2];
#pragma unroll
      for (int i = 0; i < MI2; ++i) {
        a[i][0] = As[Cfg::ai(am0 + i * 16, k0 + t)];
        a[i][1] = As[Cfg::ai(am0 + i * 16 + 8, k0 + t)];
        a[i][2] = As[Cfg::ai(am0 + i * 16, k0 + t + 4)];
        a[i][3] = As[Cfg::ai(am0 + i * 16 + 8, k0 + t + 4)];
      }
#pragma unroll
      for (int j = 0; j < Cfg::NJ; ++j) {
        b[j][0] = Bs[Cfg::bi(k0 + t, bn0 + j * 8)];
        b[j][1] = Bs[Cfg::bi(k0 + t + 4, bn0 + j * 8)];
      }
      if (nx < nk) ap.stage_part(As_nx, nx, k8, BK / 8);
#pragma unroll
      for (int i = 0; i < MI2; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j)
          mma16x8x8(acc[2 * i][j][0], acc[2 * i][j][1], acc[2 * i + 1][j][0], acc[2 * i + 1][j][1], a[i][0], a[i][1],
                    a[i][2], a[i][3], b[j][0], b[j][1]);
    }
    } else {
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
      // the A producer's work for the next stage is spread over the k4 slices,
      // so operator-tile evaluation interleaves with this slice's DMMAs
      if (nx < nk) ap.stage_part(As_nx, nx, k4, BK / 4);
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
    }
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
}

// Entries [e0, e1) of a producer's E per-thread entries handled in `part` of
// `nparts`, grouped CHUNK at a time (independent evaluations in flight
// together) and issued at the last slice of each chunk's window.
template <int E, int CHUNK>
__device__ __forceinline__ void chunk_range(int part, int nparts, int& e0, int& e1) {
  if (nparts <= 1) { e0 = 0; e1 = E; return; }
  const int csz = (E + nparts - 1) / nparts > CHUNK ? (E + nparts - 1) / nparts : CHUNK;  // entries per chunk
  const int nch = (E + csz - 1) / csz;
  const int per = nparts / nch;                      // slices per chunk window (>= 1)
  const int ch = part / per;
  if (part % per != per - 1 || ch >= nch) { e0 = e1 = 0; return; }
  e0 = ch * csz;
  e1 = (ch + 1) * csz < E ? (ch + 1) * csz : E;
}

// Adapter giving a whole-stage producer the stage_part interface (work done at part 0).
template <class P>
struct WholeStage {
  P& p;
  __device__ __forceinline__ void stage(double* s, int ks) { p.stage(s, ks); }
  __device__ __forceinline__ void stage_part(double* s, int ks, int part, int) {
    if (part == 0) p.stage(s, ks);
  }
  __device__ __forceinline__ void prefetch(int) {}
};

// Copy a (rows x cols) tile of a row-major global matrix, contiguous along
// cols, into shared memory at dst[r * sstride + c] (r < rows, c < cols),
// zero-filling outside (rlim, clim). Row r's global row is rowmap(r).
// 16-byte cp.async when `vec2` (even ld / offsets, 16B-aligned base).
// `free_dim` (1: cols, 2: rows): the dimension that is not the product's k
// dimension; entries beyond its limit feed only outputs that are never
// stored and are left untouched instead of zero-filled (see producer_copy in
// dense.cu for the measurement).
template <int NT, class RowMap>
__device__ __forceinline__ void tile_copy(double* dst, int sstride, const double* src, int64_t ld, int rows, int cols,
                                          int r0, int c0, int rlim, int clim, RowMap rowmap, bool vec2,
                                          int free_dim = 0) {
  if (vec2) {
    const int half = cols >> 1;
    for (int e = threadIdx.x; e < rows * half; e += NT) {
      int r = e / half, c = (e - r * half) * 2;
      int gr = r0 + r, gc = c0 + c;
      double* d = dst + r * sstride + c;
      if (free_dim == 2 && gr >= rlim) continue;
      if (free_dim == 1 && gc >= clim) continue;
      if (gr < rlim && gc + 1 < clim) {
        cp_async16(d, src + (int64_t)rowmap(gr) * ld + gc, true);
      } else {
        bool ok = gr < rlim && gc < clim;
        cp_async8(d, ok ? (const void*)(src + (int64_t)rowmap(gr) * ld + gc) : (const void*)src, ok);
        if (free_dim != 1 || gr >= rlim) cp_async8(d + 1, src, false);   // a k row past the end is zero in both halves
      }
    }
  } else {
    for (int e = threadIdx.x; e < rows * cols; e += NT) {
      int r = e / cols, c = e - r * cols;
      int gr = r0 + r, gc = c0 + c;
      if (free_dim == 2 && gr >= rlim) continue;
      if (free_dim == 1 && gc >= clim) continue;
      bool ok = gr < rlim && gc < clim;
      cp_async8(dst + r * sstride + c, ok ? (const void*)(src + (int64_t)rowmap(gr) * ld + gc) : (const void*)src, ok);
    }
  }
}

struct IdentityRows {
  __device__ __forceinline__ int operator()(int r) const { return r; }
};
struct MappedRows {
  const int32_t* map;
  __device__ __forceinline__ int operator()(int r) const { return map[r]; }
};

}  // namespace ublr
