// Bulk asynchronous copies (TMA, cp.async.bulk, SASS UBLKCP) global -> shared with mbarrier completion.
// One-dimensional bulk copies need no tensor map: a contiguous run of >= 16 B (16-B aligned at both
// ends) lands in shared memory and its byte count is credited to an mbarrier (complete_tx).  The
// consumer waits on the barrier's phase parity.
#pragma once
#include "common.cuh"

DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

DEV void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
// Arrive once on the barrier and add `bytes` to the transaction count of its current phase.
DEV void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Orders this thread's earlier generic-proxy shared-memory accesses before later async-proxy (TMA)
// accesses of the same memory.
DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// bytes: multiple of 16; src, dst 16-B aligned.
DEV void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
