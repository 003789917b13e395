// TMA bulk copies (cp.async.bulk, non-tensor): global -> shared completing on
// an mbarrier transaction count, shared -> global through a bulk group.  One
// issuing thread moves a whole replay slot with no register staging.
#pragma once
#include "common.cuh"

namespace dqn {

static __device__ __forceinline__ uint32_t bc_smem(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

static __device__ __forceinline__ void bc_mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bc_smem(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

static __device__ __forceinline__ void bc_mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BC_WAIT_%=;\n}" ::"r"(bc_smem(bar)),
      "r"(parity)
      : "memory");
}

// global [src, src + bytes) -> shared dst (bytes % 16 == 0, 16-B aligned),
// then shared -> global dst2; returns when the global writes are complete
static __device__ __forceinline__ void bulk_copy_via_smem(void *smem, uint64_t *bar,
                                                          const void *src, void *dst,
                                                          uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bc_smem(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(bc_smem(smem)),
      "l"(src), "r"(bytes), "r"(bc_smem(bar))
      : "memory");
  bc_mbar_wait(bar, 0);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(bc_smem(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the frame gathers use the bulk-copy engine (measured +0.3 % device / +1 %
// end to end over register copies); the register path remains for slots
// that are not 16-byte multiples
inline bool tma_gather_enabled() { return true; }

}  // namespace dqn
