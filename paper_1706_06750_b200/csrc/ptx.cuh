// ptx.cuh — thin inline-PTX wrappers for sm_100a: mbarrier, 1-D bulk async copies (TMA engine), fast reciprocal.
#pragma once
#include <stdint.h>

namespace kz {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float frcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// KZ_WAIT_SLEEP=1: the try-wait carries a suspend-time hint, so waiting threads sleep until the phase completes
// instead of re-issuing the loop.  Measured for the scale-space kernels (cond, AOS columns and rows, whose CTAs
// wait once per tile or strip): no change (1862 vs 1861 img/s; cond 20.2 vs 20.1 ms), so the default spins; the
// matcher, whose issuer and epilogue wait on every tile, uses mbar_wait_sleep.
#ifndef KZ_WAIT_SLEEP
#define KZ_WAIT_SLEEP 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if KZ_WAIT_SLEEP
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KZ_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra KZ_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KZ_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KZ_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// The same on a shared-window address computed once (hot loops: no generic → shared conversion per wait).
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KZ_WAITU_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KZ_WAITU_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// With a suspend-time hint: the waiting thread sleeps until the phase completes (or the hint elapses) instead of
// re-issuing the try-wait loop, so a waiting warp gives its issue slots to the warps that do the work.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KZ_WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra KZ_WAITS_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Global → shared bulk copy through the TMA engine; completes `bytes` on the mbarrier.  bytes % 16 == 0,
// both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 3-D tiled tensor copy global → shared through the TMA engine (box and strides in the tensor map, out-of-bounds
// elements zero-filled); completes the whole box's bytes on the mbarrier.  dst 128-byte aligned.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Shared → global 3-D tiled tensor store (out-of-bounds box elements are not written), its bulk-group commit and
// the wait until the shared source has been read (the CTA must not retire its shared memory before).  The writing
// threads make their shared stores visible to the async proxy with fence_proxy_async_smem() before the barrier
// that precedes the store.
__device__ __forceinline__ void tma_store_3d(const void* tmap, int c0, int c1, int c2, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tmap),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
    asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace kz
