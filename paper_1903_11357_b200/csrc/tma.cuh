// tma.cuh — bulk asynchronous copies global -> shared (cp.async.bulk, the non-tensor TMA path) with
// mbarrier completion tracking: the sm_100a way to keep tens of KB per SM in flight for streaming
// kernels without spending registers on it.
#pragma once
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// order prior generic-proxy shared accesses before subsequent async-proxy writes to the same buffer
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// L2 policy for streamed operator data (read once per sweep): evict first, so the vectors the kernels
// gather (x, z, p, r) stay resident in the 126 MB L2
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// evict last: operator data that is read again soon (the local solve's forward/backward turnaround)
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// one bulk copy (size multiple of 16, both addresses 16-byte aligned); completion counted on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  bulk_g2s(dst, src, bytes, bar, l2_evict_first());
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// producer-side wait: back off between polls. A producer lane that waits for its consumers to release a
// ring slot otherwise spins YIELD / TRYWAIT / BRA at full issue rate on a scheduler it shares with consumer
// warps (ncu on k_local_mrhs_r, config 3: 34% of all executed warp instructions were this loop).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t phase, unsigned ns = 128) {
  while (!mbar_try_wait(bar, phase)) __nanosleep(ns);
}
// Per translation unit: back-off of the streaming kernels' producer lanes (0 = plain spin), set from
// DGAS_PRODUCER_NS by tma_set_backoff() in the unit's setup code.
static __constant__ unsigned c_producer_ns = 0;
__device__ __forceinline__ void mbar_wait_producer(uint64_t* bar, uint32_t phase) {
  const unsigned ns = c_producer_ns;
  if (ns) mbar_wait_backoff(bar, phase, ns);
  else mbar_wait(bar, phase);
}
#ifdef TMA_HOST_BACKOFF
#include <cstdlib>
static inline void tma_set_backoff(unsigned dflt) {
  unsigned ns = dflt;
  if (const char* e = std::getenv("DGAS_PRODUCER_NS")) ns = (unsigned)std::atoi(e);
  cudaMemcpyToSymbol(c_producer_ns, &ns, sizeof(ns));
}
#endif
// load `bytes` (multiple of 16) possibly larger than the 1 MB bulk limit: chunks of 64 KB
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  mbar_expect_tx(bar, bytes);
  const uint32_t CH = 65536;
  for (uint32_t o = 0; o < bytes; o += CH) {
    uint32_t n = bytes - o < CH ? bytes - o : CH;
    bulk_g2s((char*)dst + o, (const char*)src + o, n, bar, pol);
  }
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  bulk_load(dst, src, bytes, bar, l2_evict_first());
}

// plain arrive (count 1) on an mbarrier
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier among `count` threads (multiple of 32) with id `id` (1..15)
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
