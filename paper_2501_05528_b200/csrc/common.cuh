// Shared device helpers for the uBLR B200 kernels (sm_100a, fp64).
//
// FP64 matrix math on sm_100a: tcgen05.mma has no f64 kind, so the dense
// stages use mma.sync m8n8k4 f64 (SASS DMMA.8x8x4). Measured on this pool's
// B200 (profiles/fp64_peak_r01.txt): DMMA 37.1 TFLOP/s, DFMA 36.5 TFLOP/s.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/ublr_b200.h"

namespace ublr {

// ---------------------------------------------------------------------------
// Error plumbing: C-ABI functions return UBLR_OK or a negative status and
// leave a message retrievable with ublr_last_error().
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);

#define UBLR_REQUIRE(cond, code, msg)                 \
  do {                                                \
    if (!(cond)) {                                    \
      ::ublr::set_error(msg);                         \
      return (code);                                  \
    }                                                 \
  } while (0)

#define UBLR_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::ublr::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +       \
                        " at " __FILE__ ":" + std::to_string(__LINE__));             \
      return UBLR_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define UBLR_LAUNCH_CHECK() UBLR_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// mma.sync m8n8k4 f64: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment ownership (lane = 4*g + t): a = A[g][t], b = B[t][g],
// d0 = D[g][2t], d1 = D[g][2t+1].
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// D(16x8) += A(16x8) B(8x8), fp64 (DMMA, 8x fewer instructions than m8n8k4
// for the same work). Lane (g, t): a0 = A[g][t], a1 = A[g+8][t],
// a2 = A[g][t+4], a3 = A[g+8][t+4]; b0 = B[t][g], b1 = B[t+4][g];
// d0, d1 = D[g][2t, 2t+1]; d2, d3 = D[g+8][2t, 2t+1].
__device__ __forceinline__ void mma16x8x8(double& d0, double& d1, double& d2, double& d3, double a0, double a1,
                                          double a2, double a3, double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(d0), "+d"(d1), "+d"(d2), "+d"(d3)
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// ---------------------------------------------------------------------------
// Fast fp64 log for kernel evaluation: x = 2^e * f, f in [1,2);
// f = c_j (1 + t) with c_j = 1 + (j + 1/2)/128 on the top 7 mantissa bits,
// |t| < 2^-8; log(1+t) by a degree-8 Taylor/Horner polynomial
// (truncation < 2^-72). Tables log(c_j), 1/c_j live in shared memory.
// Accuracy: ~1-2 ulp (checked against numpy in tests/test_kernels_gpu.py).
// ---------------------------------------------------------------------------
struct LogTables {
  double logc[128];
  double invc[128];
};

__device__ __forceinline__ void init_log_tables(LogTables* t) {
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    double c = 1.0 + (j + 0.5) / 128.0;
    t->logc[j] = log(c);
    t->invc[j] = 1.0 / c;
  }
}

__device__ __forceinline__ double fast_log(double x, const LogTables* tb) {
  long long bits = __double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  int j = (int)((bits >> 45) & 0x7f);
  double f = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  // c = 1 + (j + 0.5) / 128 = 1 + (2j + 1) 2^-8, built from bits (no FP64 op)
  double c = __longlong_as_double(0x3ff0000000000000LL | ((long long)(2 * j + 1) << 44));
  double t = (f - c) * tb->invc[j];
  // log(1+t) = t - t^2/2 + t^3/3 - ... (8 terms)
  double p = -1.0 / 8.0;
  p = fma(p, t, 1.0 / 7.0);
  p = fma(p, t, -1.0 / 6.0);
  p = fma(p, t, 1.0 / 5.0);
  p = fma(p, t, -1.0 / 4.0);
  p = fma(p, t, 1.0 / 3.0);
  p = fma(p, t, -1.0 / 2.0);
  p = p * t * t + t;
  const double LN2_HI = 6.93147180369123816490e-01;
  const double LN2_LO = 1.90821492927058770002e-10;
  double ed = (double)e;
  return fma(ed, LN2_HI, tb->logc[j]) + fma(ed, LN2_LO, p);
}

}  // namespace ublr
