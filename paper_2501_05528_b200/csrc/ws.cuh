// Warp-specialisation helpers: mbarrier producer/consumer rings and
// register re-balancing between warp roles (sm_90+ PTX, used on sm_100a).
//
// A ring slot s has two mbarriers: full[s] (producers -> consumers: the
// stage's operand tiles are in shared memory) and empty[s] (consumers ->
// producers: the stage has been read). Use u = ks / STAGES of slot s waits
// full[s] with parity (u & 1) and empty[s] with parity ((u & 1) ^ 1) — a
// fresh barrier reports the phase "before" phase 0 as complete, so the first
// producer pass does not block.
#pragma once
#include <cstdint>

namespace ublr {
namespace ws {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// arrive with release semantics at CTA scope (orders this thread's prior
// shared-memory writes and reads before the phase completes)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// arrive once all prior cp.async of this thread have landed (counts toward
// the expected arrivals: .noinc)
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// named barrier over `nthreads` threads (multiple of 32), id 1..15
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- thread-block clusters: the CTAs of a cluster share generated operand
// tiles through distributed shared memory. A peer's copy of a shared-memory
// object lives at mapa(own address, peer rank); stores and mbarrier arrivals
// on it use the shared::cluster window, waits stay on the CTA's own barrier
// with cluster-scope acquire.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Asynchronous 8-byte store into a peer CTA's shared memory that signals
// complete_tx(8) on an mbarrier of that peer (both addresses in the
// shared::cluster window, same CTA). The data become visible to the threads
// that observe the barrier's phase complete -- no fence on either side.
__device__ __forceinline__ void st_async_f64(uint32_t cluster_addr, double v, uint32_t cluster_mbar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(cluster_addr),
               "d"(v), "r"(cluster_mbar)
               : "memory");
}
// arrive on the CTA's own barrier and add `bytes` to the transaction count the phase waits for
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// arrive on a barrier of a peer CTA ("this warp has finished reading the
// stage"): the reads it orders are complete when the arrive issues (their
// values fed instructions issued before it), so CTA-scope release suffices
// and no cluster-scope fence is emitted
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// every thread of every CTA of the cluster
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

}  // namespace ws
}  // namespace ublr
