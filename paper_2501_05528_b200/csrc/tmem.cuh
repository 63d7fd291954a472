// Tensor memory (TMEM) as accumulator storage for fp64 CUDA-core / DMMA
// kernels on sm_100a.
//
// tcgen05.mma has no f64 kind, but the 256 KB of TMEM per SM is still there:
// tcgen05.st / tcgen05.ld move 32-bit columns between a warp's registers and
// its 32-lane quarter of TMEM (warp w addresses lanes 32*(w%4) .. +31).
// The tagged sketch keeps ell-fold accumulators there that do not fit in
// registers.
#pragma once
#include <cstdint>

namespace ublr {
namespace tmem {

// One warp allocates `ncols` columns (power of two, 32..512) and writes the
// base address to *slot (shared memory).
__device__ __forceinline__ void alloc(uint32_t* slot, uint32_t ncols) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(slot));
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 8 doubles (16 x 32-bit columns) per lane.
__device__ __forceinline__ void st8(uint32_t taddr, const double (&v)[8]) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[2 * i] = static_cast<uint32_t>(__double2loint(v[i]));
    r[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v[i]));
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void ld8(uint32_t taddr, double (&v)[8]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  wait_ld();
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double(static_cast<int>(r[2 * i + 1]), static_cast<int>(r[2 * i]));
}

// 16 x 32-bit columns per lane without waiting: issue several, then one
// wait_ld(), then unpack with unpack8 (hides the TMEM load latency once per
// batch instead of once per load).
__device__ __forceinline__ void ld8_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void unpack8(const uint32_t (&r)[16], double (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double(static_cast<int>(r[2 * i + 1]), static_cast<int>(r[2 * i]));
}

// address of (lane base of this warp's quarter, column)
__device__ __forceinline__ uint32_t addr(uint32_t base, int warp, int col) {
  return base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(col);
}

}  // namespace tmem
}  // namespace ublr
