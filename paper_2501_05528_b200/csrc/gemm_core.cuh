// Shared fp64 DMMA main loop for the operator-apply and batched GEMM kernels.
//
// CTA tile BM x BN, k-step BK, WMW x WNW warps, each warp owning a
// (BM/WMW) x (BN/WNW) tile of m8n8k4 accumulators. Operand tiles live in
// shared memory k-major (As[k][m], Bs[k][n]) with a +4 double pad, so the
// fragment loads (lane (g, t) reads As[k0+t][m0+g]) are conflict-free.
// A STAGES-deep ring of shared buffers lets the producers (cp.async for
// stored operands, in-register generation for operator tiles) fill stage
// ks+STAGES-1 while the tensor pipe consumes stage ks; the fragments of the
// next k4 slice are loaded before the current slice's DMMAs issue.
#pragma once
#include "common.cuh"

namespace ublr {

template <int BM_, int BN_, int BK_, int WMW_, int WNW_, int STAGES_>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WMW = WMW_, WNW = WNW_, STAGES = STAGES_;
  static constexpr int NT = WMW * WNW * 32;
  static constexpr int SA = BM + 4;
  static constexpr int SB = BN + 4;
  static constexpr int WM = BM / WMW;
  static constexpr int WN = BN / WNW;
  static constexpr int MI = WM / 8;
  static constexpr int NJ = WN / 8;
  static constexpr int A_STAGE = BK * SA;  // doubles
  static constexpr int B_STAGE = BK * SB;
  static constexpr size_t smem_bytes() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double); }
};

// acc += A_tile * B_tile over nk k-steps. Producers fill one stage:
//   ap.stage(double* As /*[BK][SA]*/, int ks);  bp.stage(double* Bs /*[BK][SB]*/, int ks)
// and may issue cp.async; one commit group per stage is made here.
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
    {
      int nx = ks + STAGES - 1;
      int slot = nx % STAGES;
      if (nx < nk) {
        ap.stage(As0 + slot * Cfg::A_STAGE, nx);
        bp.stage(Bs0 + slot * Cfg::B_STAGE, nx);
      }
      cp_async_commit();
    }
    const double* As = As0 + (ks % STAGES) * Cfg::A_STAGE;
    const double* Bs = Bs0 + (ks % STAGES) * Cfg::B_STAGE;
    double a[2][Cfg::MI], b[2][Cfg::NJ];
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i) a[0][i] = As[t * Cfg::SA + am0 + i * 8];
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j) b[0][j] = Bs[t * Cfg::SB + bn0 + j * 8];
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int cur = k4 & 1;
      if (k4 + 1 < BK / 4) {
        const int kr = (k4 + 1) * 4 + t;
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i) a[cur ^ 1][i] = As[kr * Cfg::SA + am0 + i * 8];
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) b[cur ^ 1][j] = Bs[kr * Cfg::SB + bn0 + j * 8];
      }
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) mma8x8x4(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
    }
  }
  cp_async_wait<0>();
}

}  // namespace ublr
