// match.cu — brute-force descriptor matching (reading A25) on the 5th-generation tensor
// cores: the one dense contraction of the method, desc_A · desc_Bᵀ.
//
//   1. k_match_prep: fp32 [n][64] → fp16 rows in the UMMA K-major SWIZZLE_128B layout, pre-tiled by kTileR = 128
//      rows (each 16 KB tile is the exact shared-memory image, so one 1-D TMA bulk copy stages it), a 128-bit validity
//      mask per tile (degenerate = all-zero descriptors and padding rows are never candidates) and the norm
//      range of the valid rows.
//   2. k_match_topk: one CTA per 128 query rows and reference part (the reference range is split into up to
//      kMaxSplit parts when the query blocks alone cannot fill two CTAs per SM).  A TMA warp streams the reference
//      tiles through a kStages = 3 mbarrier ring, one thread issues tcgen05.mma kind::f16 (M = 128, N = 128,
//      K = 4 x 16) into a double-buffered TMEM accumulator (2 x 128 columns), and 8 epilogue warps drain it with
//      tcgen05.ld (warp w reads TMEM lanes 32·(w%4).. = its 32 query rows, column half w/4), keeping each row's
//      eight best approximate scores per part.  Per 32-column chunk: the chunk maximum against each row's 8th best
//      (the larger of its own column group's and the other group's, published once per tile); rows with candidates
//      build a mask from the sign bits of thr − v; one candidate per row is the chunk maximum, inserted from
//      registers; more go through shared memory.  All mbarrier waits sleep (suspend-time hint) instead of spinning.  fp16 operands (descriptor components lie in [−1, 1]; fp16 has bf16's tensor rate and
//      3 more significand bits), fp32 accumulation: |s_approx − a·b| <= 2^-10·|a||b| + accumulation slack.
//   3. k_match_rerank: one warp per query: exact fp32 distances ||a − b|| for the eight candidates, ordered by
//      (distance, index).  The result is CERTIFIED exact when the second candidate distance is below the
//      smallest distance any non-candidate can have, |a|² + min|b|² − 2(s_8 + ε); otherwise the warp scans every
//      reference exactly (rare).  With a split range the parts' top-8 lists are merged here, and the certificate
//      bound uses the largest part-wise 8th score.  So tensor cores do the bulk and the decision is the exact fp32 one.
//   4. k_match_final: ratio test d1 < ratio·d2 and the symmetric cross-check from the reverse pass.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "kaze_internal.cuh"
#include "ptx.cuh"

namespace kz {

namespace {

constexpr int kTileR = 128;                 // reference rows per tile (UMMA N); 128 lets two CTAs share an SM's TMEM
constexpr int kTileQ = 128;                 // query rows per CTA (UMMA M)
constexpr int kTileBytes = kTileR * 128;    // 64 fp16 = 128 B per row
constexpr int kStages = 3;  // reference-tile ring depth (TMA → MMA)
constexpr int kMaxSplit = 4;  // reference-range parts per query block when the query blocks alone cannot fill the GPU
constexpr int kCand = 8;  // approximate candidates kept per query (4: 1400 of 15.8k KAZE rows uncertified, 3.4 ms)
// KZ_MATCH_DEEP: one CTA per SM with a 4-deep ring of whole-tile accumulators (all 512 TMEM columns) and 16
// epilogue warps on column quarters, instead of two CTAs per SM with 2-deep rings and 8 warps each.
#ifndef KZ_MATCH_DEEP
#define KZ_MATCH_DEEP 0
#endif
constexpr int kCtasPerSm = KZ_MATCH_DEEP ? 1 : 2;
constexpr int kEpiWarps = KZ_MATCH_DEEP ? 16 : 8;  // 4 TMEM lane groups x column groups (round 1, 2 CTAs/SM: 16 warps with column quarters 3.64 vs 3.59 ms at 65536^2)
constexpr int kColGroups = kEpiWarps / 4;
#ifndef KZ_MATCH_SHARE_THR
#define KZ_MATCH_SHARE_THR 1
#endif
#ifndef KZ_MATCH_SLEEP
#define KZ_MATCH_SLEEP 1
#endif
#ifndef KZ_MATCH_ONELD
#define KZ_MATCH_ONELD 1
#endif
#ifndef KZ_MATCH_SIGNMASK
#define KZ_MATCH_SIGNMASK 1
#endif
constexpr int kThreads = (kEpiWarps + 2) * 32;  // + TMA warp + MMA warp
// Accumulator stages: each reference tile is accumulated as kHalves column slices of kAccW columns (N = kAccW MMAs),
// in a ring of kAcc = 2·kHalves TMEM stages (256 columns per CTA either way).  Finer slices let the MMA run further
// ahead of the epilogue: with whole-tile stages (kHalves = 1) the issuer waited on a free accumulator for every tile
// and the epilogue on a full one (ncu, 65536^2: 60-70 try-wait spins per tile in the issuer, ~10 per warp and tile in
// the epilogue).
#ifndef KZ_MATCH_HALVES
#define KZ_MATCH_HALVES 1
#endif
constexpr int kHalves = KZ_MATCH_HALVES;
constexpr int kAccW = kTileR / kHalves;
constexpr int kAcc = (KZ_MATCH_DEEP ? 4 : 2) * kHalves;
constexpr float kEps = 1.0f / 1024.0f + 2e-5f;  // fp16 rounding of both operands (2·2^-11) + fp32 sum slack

// ---- tcgen05 / mbarrier wrappers (PTX ISA 8.7, sm_100a) ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 columns of 32-bit accumulators → 32 registers per thread (thread i ↔ lane base+i).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: rows of 128 B, 8-row atoms 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor kind::f16: D f32 (bits 4-5 = 1), A/B f16 (format 0 at bits 7-9 / 10-12), both K-major,
// N = kTileR (bits 17-22 = N/8), M = 128 (bits 24-28 = M/16).
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(kAccW >> 3) << 17) | ((uint32_t)(kTileQ >> 4) << 24);

__global__ void __launch_bounds__(256) k_match_prep(const float* __restrict__ D, int n, int ntiles,
                                                    uint8_t* __restrict__ tiles, uint32_t* __restrict__ valid,
                                                    unsigned* __restrict__ norm_range /* [min bits, max bits] */) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte chunk (8 values) per thread
    const int r = g >> 3, c = g & 7;
    if (r >= ntiles * kTileR) return;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (r < n) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(D + (size_t)r * 64 + 8 * c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(D + (size_t)r * 64 + 8 * c + 4));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    const int t = r / kTileR, rr = r - t * kTileR;
    uint4* dst = reinterpret_cast<uint4*>(tiles + (size_t)t * kTileBytes + rr * 128 + ((c ^ (rr & 7)) << 4));
    *dst = make_uint4(w[0], w[1], w[2], w[3]);
    // row norm² from the 8 lanes of the row (lanes 8q..8q+7 of a warp)
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s = fmaf(v[i], v[i], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    const bool ok = r < n && s > 0.f;
    const unsigned bits = __ballot_sync(0xffffffffu, ok && c == 0);
    if ((threadIdx.x & 31) == 0) {
        // the warp covers rows 4·(g/32) .. +3: bits 0, 8, 16, 24 of the ballot
        const uint32_t nib = ((bits >> 0) & 1u) | ((bits >> 7) & 2u) | ((bits >> 14) & 4u) | ((bits >> 21) & 8u);
        const int r0 = r;  // lane 0's row (c == 0)
        if (nib) atomicOr(valid + (r0 >> 5), nib << (r0 & 31));
    }
    if (c == 0 && ok) {
        const float nr = sqrtf(s);
        atomicMin(norm_range, __float_as_uint(nr));  // positive floats order as unsigned
        atomicMax(norm_range + 1, __float_as_uint(nr));
    }
}

// Producer / MMA-issuer waits (one thread each): suspended rather than spinning (KZ_MATCH_SLEEP).
__device__ __forceinline__ void kwait(uint64_t* bar, uint32_t parity) {
#if KZ_MATCH_SLEEP
    mbar_wait_sleep(smem_u32(bar), parity);
#else
    mbar_wait(bar, parity);
#endif
}

struct TopK {
    float s[kCand];
    int j[kCand];
};

// Sorted insertion as a fixed compare-exchange chain (no runtime indexing, so the list stays in registers).
// Order: higher score first; on equal scores the lower index first.
__device__ __forceinline__ void topk_push(TopK& t, float v, int j) {
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        const bool sw = v > t.s[q] || (v == t.s[q] && j < t.j[q]);
        const float ts = t.s[q];
        const int tj = t.j[q];
        t.s[q] = sw ? v : ts;
        t.j[q] = sw ? j : tj;
        v = sw ? ts : v;
        j = sw ? tj : j;
    }
}
// Scan-time insertion: columns arrive in increasing j, so "higher score first" alone already keeps the earlier of
// equal scores; no index comparisons (5 instead of 8 instructions per stage).
__device__ __forceinline__ void topk_push_scan(TopK& t, float v, int j) {
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        const bool sw = v > t.s[q];
        const float ts = t.s[q];
        const int tj = t.j[q];
        t.s[q] = sw ? v : ts;
        t.j[q] = sw ? j : tj;
        v = sw ? ts : v;
        j = sw ? tj : j;
    }
}
__device__ __forceinline__ void topk_insert(TopK& t, float v, int j) {
    if (v > t.s[kCand - 1]) topk_push_scan(t, v, j);
}

__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_match_topk(const uint8_t* __restrict__ Qt, int nq,
                                                            const uint8_t* __restrict__ Rt, int nr,
                                                            const uint32_t* __restrict__ rvalid,
                                                            float* __restrict__ cand_s, int* __restrict__ cand_j) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the swizzle atoms
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                    // 16 KB
    uint8_t* sB = smem + kTileQ * 128;     // kStages x 16 KB
    __shared__ __align__(8) uint64_t bar_full[kStages], bar_empty[kStages], bar_acc_full[kAcc], bar_acc_empty[kAcc], bar_a;
    __shared__ uint32_t tmem_base_slot;
#if KZ_MATCH_SHARE_THR
    // each column group's current 8th-best score per query row, published once per tile: a column group filters with
    // the larger of its own and the other groups' (a score at or below another group's 8th best has 8 scores at
    // least as high elsewhere, so dropping it keeps every non-candidate at or below the merged list's 8th score —
    // what the re-rank certificate assumes).  Stale values are smaller, so they are safe too.
    __shared__ float thr_sh[kColGroups][kTileQ];
    for (int i = threadIdx.x; i < kColGroups * kTileQ; i += blockDim.x) (&thr_sh[0][0])[i] = -INFINITY;
#endif
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this CTA scans reference tiles [tb, tb + ntiles) — part blockIdx.y of gridDim.y — and writes its own top-8
    const int ntiles_all = (nr + kTileR - 1) / kTileR;
    const int tb = (int)((long long)ntiles_all * blockIdx.y / gridDim.y);
    const int ntiles = (int)((long long)ntiles_all * (blockIdx.y + 1) / gridDim.y) - tb;
    Rt += (size_t)tb * kTileBytes;
    rvalid += (size_t)tb * (kTileR / 32);
    cand_s += (size_t)blockIdx.y * nq * kCand;
    cand_j += (size_t)blockIdx.y * nq * kCand;
    const int q0 = blockIdx.x * kTileQ;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&bar_full[i], 1);
            mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            mbar_init(&bar_acc_full[i], 1);
            mbar_init(&bar_acc_empty[i], kEpiWarps * 32);
        }
        mbar_init(&bar_a, 1);
        fence_mbar_init();
    }
    if (warp == kEpiWarps + 1) tmem_alloc(&tmem_base_slot, kAcc * kAccW);  // the accumulator ring (256 columns)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_slot;

    if (warp == kEpiWarps) {  // ===== TMA producer =====
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar_a, kTileQ * 128);
            bulk_g2s(sA, Qt + (size_t)q0 * 128, kTileQ * 128, &bar_a);
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % kStages;
                if (t >= kStages) kwait(&bar_empty[s], ((t / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&bar_full[s], kTileBytes);
                bulk_g2s(sB + s * kTileBytes, Rt + (size_t)t * kTileBytes, kTileBytes, &bar_full[s]);
            }
        }
    } else if (warp == kEpiWarps + 1) {  // ===== MMA issuer (one thread) =====
        if (lane == 0) {
            mbar_wait(&bar_a, 0);
            const uint32_t a_addr = smem_u32(sA);
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % kStages;
                kwait(&bar_full[s], (t / kStages) & 1);
#pragma unroll
                for (int hh = 0; hh < kHalves; ++hh) {
                    const int u = t * kHalves + hh, st = u % kAcc;
                    if (u >= kAcc) kwait(&bar_acc_empty[st], ((u / kAcc) - 1) & 1);
                    tc_fence_after();
                    // reference rows hh·kAccW.. of the tile: whole 8-row swizzle atoms, kAccW·128 B further on
                    const uint32_t b_addr = smem_u32(sB + s * kTileBytes) + hh * kAccW * 128;
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // K = 64 = 4 x 16, +32 B along the swizzled row per step
                        mma_f16(tmem + st * kAccW, smem_desc_sw128(a_addr + 32 * k), smem_desc_sw128(b_addr + 32 * k),
                                kIdesc, k > 0 ? 1u : 0u);
                    mma_commit(&bar_acc_full[st]);  // accumulator stage ready for the epilogue
                }
                mma_commit(&bar_empty[s]);  // smem stage free once these MMAs are done
            }
        }
    } else {  // ===== epilogue warps: TMEM → registers → running top-8 (kCand) per query row =====
        const int g = warp & 3, h = warp >> 2;  // TMEM lane group (query rows 32g..), column group
        float* sv = reinterpret_cast<float*>(sB + kStages * kTileBytes) + warp * 32 * 32;  // 4 KB per epilogue warp
        TopK tk;
#pragma unroll
        for (int q = 0; q < kCand; ++q) {
            tk.s[q] = -INFINITY;
            tk.j[q] = -1;
        }
        constexpr int kChunks = kAccW / kColGroups / 32;  // 32-column chunks per warp and accumulator stage
        float thr_other = -INFINITY;  // the other column groups' published 8th best for this lane's row
        // loop-invariant addresses (the per-tile code re-derived them from the generic pointers: ~1/3 of its
        // instructions)
        const uint32_t acc_full0 = smem_u32(&bar_acc_full[0]), acc_empty0 = smem_u32(&bar_acc_empty[0]);
        const uint32_t tmem_row = tmem + ((uint32_t)(32 * g) << 16) + (uint32_t)(h * (kAccW / kColGroups));
        const uint32_t* rv = rvalid + ((h * (kAccW / kColGroups)) >> 5);
#if KZ_MATCH_SHARE_THR
        // relaxed CTA-scope accesses: the publication is unordered by design (any value seen is a valid bound), and
        // relaxed atomics make that explicit instead of a data race
        const uint32_t thr_mine = smem_u32(&thr_sh[h][32 * g + lane]);
        const uint32_t thr_col = smem_u32(&thr_sh[0][32 * g + lane]);
#endif
        for (int u = 0; u < ntiles * kHalves; ++u) {
            const int t = u / kHalves, hh = u - t * kHalves, st = u % kAcc;
#if KZ_MATCH_SHARE_THR
            if (hh == 0) {
                asm volatile("st.relaxed.cta.shared.f32 [%0], %1;" ::"r"(thr_mine), "f"(tk.s[kCand - 1]) : "memory");
#pragma unroll
                for (int h2 = 0; h2 < kColGroups; ++h2)
                    if (h2 != h) {
                        float o;
                        asm volatile("ld.relaxed.cta.shared.f32 %0, [%1];" : "=f"(o) : "r"(thr_col + 4u * h2 * kTileQ) : "memory");
                        thr_other = fmaxf(thr_other, o);
                    }
            }
#endif
            // the tile's validity words (32 columns each) are loaded before the accumulator wait, so their latency
            // hides behind it instead of stalling the chunk scan
            uint32_t vmk[kChunks];
#pragma unroll
            for (int ch = 0; ch < kChunks; ++ch)
                vmk[ch] = __ldg(rv + ((t * kTileR + hh * kAccW + ch * 32) >> 5));
#if KZ_MATCH_SLEEP
            mbar_wait_sleep(acc_full0 + 8 * st, (u / kAcc) & 1);
#else
            mbar_wait_u32(acc_full0 + 8 * st, (u / kAcc) & 1);
#endif
            tc_fence_after();
#if !KZ_MATCH_ONELD
            // all of this warp's chunks of the tile leave TMEM behind one wait (several loads in flight, not one)
            uint32_t vr[kChunks][32];
#pragma unroll
            for (int ch = 0; ch < kChunks; ++ch)
                tmem_ld32_nowait(tmem_row + (uint32_t)(st * kAccW + ch * 32), vr[ch]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // the accumulator is in registers now: hand it back to the MMA issuer before scanning it
            tc_fence_before();
            mbar_arrive_u32(acc_empty0 + 8 * st);
#endif
#pragma unroll
            for (int ch = 0; ch < kChunks; ++ch) {
#if KZ_MATCH_ONELD
                // one chunk in registers at a time (32 instead of 64 live values); the accumulator goes back to
                // the MMA issuer once the last chunk is loaded
                uint32_t vrc[32];
                tmem_ld32_nowait(tmem_row + (uint32_t)(st * kAccW + ch * 32), vrc);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (ch == kChunks - 1) {
                    tc_fence_before();
                    mbar_arrive_u32(acc_empty0 + 8 * st);
                }
#else
                const uint32_t (&vrc)[32] = vr[ch];
#endif
                const int col = hh * kAccW + h * (kAccW / kColGroups) + ch * 32;
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(vrc[i]);
                const int j0 = (tb + t) * kTileR + col;
                const uint32_t vm = vmk[ch];  // 32 columns = one validity word
                if (vm != 0xffffffffu) {  // warp-uniform and rare: padding / degenerate references never compete
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = ((vm >> i) & 1u) ? v[i] : -INFINITY;
                }
                // Chunk maximum first: once the lists have settled, most chunks beat no row's 8th best and cost
                // ~16 FMNMX3 instead of a per-column candidate mask.
                const float thr = fmaxf(tk.s[kCand - 1], thr_other);
                float mx = v[0];
#pragma unroll
                for (int i = 1; i < 31; i += 2) mx = fmaxf(mx, fmaxf(v[i], v[i + 1]));
                mx = fmaxf(mx, v[31]);
                if (!__any_sync(0xffffffffu, mx > thr)) continue;
                // candidate mask of this lane's row: columns scoring above its current 8th best
                uint32_t cand = 0u;
#if KZ_MATCH_SIGNMASK
                // bit i = sign of thr − v[i] (v > thr ⇔ thr − v < 0; equal scores give +0, and −inf − (−inf) the
                // positive canonical NaN): one FADD2 per column pair and one funnel shift per column, instead of a
                // compare, a select and half an add per column
#pragma unroll
                for (int i = 30; i >= 0; i -= 2) {
                    const float2 d = __fadd2_rn(make_float2(thr, thr), make_float2(-v[i], -v[i + 1]));
                    cand = __funnelshift_l(__float_as_uint(d.y), cand, 1);
                    cand = __funnelshift_l(__float_as_uint(d.x), cand, 1);
                }
                // one candidate in the row's chunk (the common case once the lists have settled) is the chunk
                // maximum itself: insert it straight from the register, without the shared-memory round trip
                if (!__any_sync(0xffffffffu, (cand & (cand - 1u)) != 0u)) {
                    if (cand) topk_push_scan(tk, mx, j0 + __ffs(cand) - 1);
                    continue;
                }
#else
#pragma unroll
                for (int i = 0; i < 32; ++i) cand |= (v[i] > thr ? 1u : 0u) << i;
#endif
                if (__any_sync(0xffffffffu, cand != 0u)) {
                    // Insert each lane's candidates in column order; the warp iterates max-over-lanes times, not
                    // once per column any lane needs (the values go through shared memory for indexed access).
#pragma unroll
                    for (int i = 0; i < 32; ++i) sv[i * 32 + lane] = v[i];
                    __syncwarp();
                    while (__any_sync(0xffffffffu, cand != 0u)) {
                        if (cand) {
                            const int i = __ffs(cand) - 1;
                            cand &= cand - 1u;
                            topk_insert(tk, sv[i * 32 + lane], j0 + i);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        // merge the column groups of each row through shared memory (the B ring is free by now)
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32));
        float* ms = reinterpret_cast<float*>(sB);
        int* mj = reinterpret_cast<int*>(sB + (kColGroups - 1) * kTileQ * kCand * sizeof(float));
        const int row = 32 * g + lane;
        if (h > 0) {
#pragma unroll
            for (int q = 0; q < kCand; ++q) {
                ms[((h - 1) * kTileQ + row) * kCand + q] = tk.s[q];
                mj[((h - 1) * kTileQ + row) * kCand + q] = tk.j[q];
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32));
        if (h == 0) {
            // the other groups' columns interleave with group 0's across tiles: merge by (score, index)
            for (int h2 = 1; h2 < kColGroups; ++h2)
#pragma unroll
                for (int q = 0; q < kCand; ++q) {
                    const int j = mj[((h2 - 1) * kTileQ + row) * kCand + q];
                    if (j >= 0) topk_push(tk, ms[((h2 - 1) * kTileQ + row) * kCand + q], j);
                }
            const int qg = q0 + row;
            if (qg < nq) {
#pragma unroll
                for (int q = 0; q < kCand; ++q) {
                    cand_s[(size_t)qg * kCand + q] = tk.s[q];
                    cand_j[(size_t)qg * kCand + q] = tk.j[q];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, kAcc * kAccW);
    }
}

// Exact fp32 distance of query a (lane holds dims 2·lane, 2·lane+1) to reference row j; butterfly sum (the same
// order in every call, so equal inputs give equal distances).
__device__ __forceinline__ float exact_d2(float2 a, const float* __restrict__ R, int j, int lane) {
    const float2 b = __ldg(reinterpret_cast<const float2*>(R + (size_t)j * 64) + lane);
    const float dx = a.x - b.x, dy = a.y - b.y;
    float s = fmaf(dx, dx, dy * dy);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// (d², j) order: smaller distance first, lower index on ties.
__device__ __forceinline__ bool before(float d, int j, float d2, int j2) { return d < d2 || (d == d2 && j < j2); }

__global__ void __launch_bounds__(256) k_match_rerank(const float* __restrict__ Q, int nq, const float* __restrict__ R,
                                                      int nr, const uint32_t* __restrict__ rvalid,
                                                      const unsigned* __restrict__ rnorm,
                                                      const float* __restrict__ cand_s, const int* __restrict__ cand_j,
                                                      int nsplit, int* __restrict__ best, float* __restrict__ d1o,
                                                      float* __restrict__ d2o, int* __restrict__ uncertified) {
    __shared__ __align__(16) float qsh[8][64];  // the query, for the lane-parallel exact scan
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= nq) return;
    const float2 a = __ldg(reinterpret_cast<const float2*>(Q + (size_t)q * 64) + lane);
    float na2 = fmaf(a.x, a.x, a.y * a.y);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) na2 += __shfl_xor_sync(0xffffffffu, na2, o);
    if (!(na2 > 0.f)) {  // degenerate query: never matched
        if (lane == 0) {
            best[q] = -1;
            d1o[q] = -1.f;
            d2o[q] = -1.f;
        }
        return;
    }
    float bd1 = INFINITY, bd2 = INFINITY;
    int bj1 = -1;
    // the largest kept-last score over the parts whose list is full: every non-candidate scores at most that
    float s8 = -INFINITY;
    bool any_full = false;
    for (int p = 0; p < nsplit; ++p) {  // parts cover disjoint reference ranges: no duplicates
        const float* ps = cand_s + ((size_t)p * nq + q) * kCand;
        const int* pj = cand_j + ((size_t)p * nq + q) * kCand;
        int ncand = 0;
#pragma unroll
        for (int c = 0; c < kCand; ++c) {
            const int j = __ldg(pj + c);
            if (j < 0) continue;
            ++ncand;
            const float d = exact_d2(a, R, j, lane);
            if (before(d, j, bd1, bj1)) {
                bd2 = bd1;
                bd1 = d;
                bj1 = j;
            } else if (d < bd2) {
                bd2 = d;
            }
        }
        if (ncand == kCand) {  // a part with fewer kept than kCand kept all its valid references
            any_full = true;
            s8 = fmaxf(s8, __ldg(ps + kCand - 1));
        }
    }
    // certification: a non-candidate has true score <= s8 + ε|a|max|b|, hence distance² >= the bound below
    bool cert = true;
    if (any_full) {
        const float bmin = __uint_as_float(rnorm[0]), bmax = __uint_as_float(rnorm[1]);
        const float na = sqrtf(na2);
        const float eps = kEps * na * bmax + 1e-5f;
        const float bound = na2 + bmin * bmin - 2.f * (s8 + eps);
        cert = bd2 < bound * (1.f - 4e-7f) - 1e-7f;
    }
    if (!cert) {  // exact scan of every valid reference (rare): lane-parallel over the references
        if (lane == 0) atomicAdd(uncertified, 1);
        float* qa = qsh[threadIdx.x >> 5];
        qa[2 * lane] = a.x;
        qa[2 * lane + 1] = a.y;
        __syncwarp();
        bd1 = INFINITY;
        bd2 = INFINITY;
        bj1 = -1;
        for (int j = lane; j < nr; j += 32) {  // each lane: its references in increasing j
            if (!((__ldg(rvalid + (j >> 5)) >> (j & 31)) & 1u)) continue;
            const float4* b4 = reinterpret_cast<const float4*>(R + (size_t)j * 64);
            float d = 0.f;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float4 b = __ldg(b4 + k);
                const float4 q = reinterpret_cast<const float4*>(qa)[k];
                const float dx = q.x - b.x, dy = q.y - b.y, dz = q.z - b.z, dw = q.w - b.w;
                d = fmaf(dx, dx, d);
                d = fmaf(dy, dy, d);
                d = fmaf(dz, dz, d);
                d = fmaf(dw, dw, d);
            }
            if (before(d, j, bd1, bj1)) {
                bd2 = bd1;
                bd1 = d;
                bj1 = j;
            } else if (d < bd2) {
                bd2 = d;
            }
        }
        // merge the lanes' (first, second) lists: first by (distance, index), second = next distance
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float od1 = __shfl_xor_sync(0xffffffffu, bd1, o), od2 = __shfl_xor_sync(0xffffffffu, bd2, o);
            const int oj1 = __shfl_xor_sync(0xffffffffu, bj1, o);
            if (oj1 >= 0 && (bj1 < 0 || before(od1, oj1, bd1, bj1))) {
                bd2 = fminf(bd1, od2);
                bd1 = od1;
                bj1 = oj1;
            } else {
                bd2 = fminf(bd2, od1);
            }
        }
    }
    if (lane == 0) {
        best[q] = bj1;
        d1o[q] = bj1 >= 0 ? sqrtf(bd1) : -1.f;
        d2o[q] = isinf(bd2) ? -1.f : sqrtf(bd2);
    }
}

__global__ void k_match_final(int na, const int* __restrict__ bestAB, const float* __restrict__ d1,
                              const float* __restrict__ d2, const int* __restrict__ bestBA, float ratio,
                              int32_t* __restrict__ match, float* __restrict__ dist, int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int j = bestAB[i];
    int m = -1;
    if (j >= 0) {
        const bool ratio_ok = d2[i] < 0.f || d1[i] < ratio * d2[i];  // d2 = ∞ (−1) passes
        if (ratio_ok && bestBA[j] == i) m = j;
    }
    match[i] = m;
    if (dist) dist[i] = d1[i];
    if (m >= 0) atomicAdd(count, 1);
}

__global__ void k_match_none(int na, int32_t* __restrict__ match, float* __restrict__ dist) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    match[i] = -1;
    if (dist) dist[i] = -1.f;
}

}  // namespace

// ---- scratch layout ----
struct MatchScratch {
    size_t tilesA, tilesB, validA, validB, normA, normB, candS, candJ, bestAB, bestBA, d1, d2, d1r, d2r, flags, total;
};

static MatchScratch match_layout(int na, int nb) {
    auto al = [](size_t v) { return (v + 1023) / 1024 * 1024; };
    const size_t ta = (size_t)((na + kTileR - 1) / kTileR), tb = (size_t)((nb + kTileR - 1) / kTileR);
    const size_t nmax = (size_t)(na > nb ? na : nb);
    MatchScratch m{};
    size_t o = 0;
    m.tilesA = o; o += al(ta * kTileBytes);
    m.tilesB = o; o += al(tb * kTileBytes);
    m.validA = o; o += al(ta * kTileR / 8);
    m.validB = o; o += al(tb * kTileR / 8);
    m.normA = o; o += al(8);
    m.normB = o; o += al(8);
    m.candS = o; o += al(nmax * kCand * kMaxSplit * sizeof(float));
    m.candJ = o; o += al(nmax * kCand * kMaxSplit * sizeof(int));
    m.bestAB = o; o += al((size_t)na * sizeof(int));
    m.bestBA = o; o += al((size_t)nb * sizeof(int));
    m.d1 = o; o += al((size_t)na * sizeof(float));
    m.d2 = o; o += al((size_t)na * sizeof(float));
    m.d1r = o; o += al((size_t)nb * sizeof(float));
    m.d2r = o; o += al((size_t)nb * sizeof(float));
    m.flags = o; o += al(16);
    m.total = o;
    return m;
}

size_t match_scratch_bytes(int na, int nb) { return match_layout(na, nb).total; }

static cudaError_t run_direction(const float* Q, int nq, const uint8_t* Qt, const float* R, int nr, const uint8_t* Rt,
                                 const uint32_t* rvalid, const unsigned* rnorm, float* cs, int* cj, int* best,
                                 float* d1, float* d2, int* unc, cudaStream_t s) {
    const int smem = kTileQ * 128 + kStages * kTileBytes + kEpiWarps * 32 * 32 * 4 + 1024;
    if (!ensure_smem_optin(reinterpret_cast<const void*>(k_match_topk), smem)) return cudaErrorInvalidValue;
    // When the query blocks alone cannot fill the two CTA slots per SM, split the reference range into nsplit parts:
    // the largest wave efficiency (CTAs / slots) / ⌈CTAs / slots⌉ over nsplit <= kMaxSplit (<= the tile count), the
    // smallest nsplit on ties (the KAZE pair, 124 query blocks: 2 parts 0.515 ms vs 3 parts 0.56).  Enough query blocks
    // are never split: each part adds 8 candidates per query to the exact re-rank (65536²: 4 parts 4.43 ms vs 3.30
    // unsplit, although 4 parts fill 6.92 of 7 waves and 1 part 1.73 of 2).
    const int qblocks = (nq + kTileQ - 1) / kTileQ, rtiles = (nr + kTileR - 1) / kTileR;
    static const int split_knob = tune_knob("KAZE_MATCH_SPLIT", 0);  // > 0 forces the part count (A/B)
    const int slots = kCtasPerSm * device_sm_count();
    int nsplit = 1;
    double best_eff = -1.0;
    for (int sp = 1; qblocks < slots && sp <= kMaxSplit && sp <= (rtiles > 0 ? rtiles : 1); ++sp) {
        const double w = (double)qblocks * sp / slots;
        const double eff = w / std::ceil(w);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            nsplit = sp;
        }
    }
    if (split_knob > 0) nsplit = std::min(std::min(split_knob, kMaxSplit), rtiles > 0 ? rtiles : 1);
    k_match_topk<<<dim3(qblocks, nsplit), kThreads, smem, s>>>(Qt, nq, Rt, nr, rvalid, cs, cj);
    k_match_rerank<<<(nq + 7) / 8, 256, 0, s>>>(Q, nq, R, nr, rvalid, rnorm, cs, cj, nsplit, best, d1, d2, unc);
    return cudaGetLastError();
}

// Returns a cudaError_t (0 on success); stats (optional, device) receives [matches, uncertified rows].
int match_run(const float* A, int na, const float* B, int nb, float ratio, int32_t* match, float* dist,
              void* scratch, size_t bytes, int* stats, cudaStream_t s) {
    const MatchScratch L = match_layout(na, nb);
    if (bytes < L.total) return -1;
    uint8_t* base = static_cast<uint8_t*>(scratch);
    uint8_t* tA = base + L.tilesA;
    uint8_t* tB = base + L.tilesB;
    uint32_t* vA = reinterpret_cast<uint32_t*>(base + L.validA);
    uint32_t* vB = reinterpret_cast<uint32_t*>(base + L.validB);
    unsigned* nA = reinterpret_cast<unsigned*>(base + L.normA);
    unsigned* nB = reinterpret_cast<unsigned*>(base + L.normB);
    int* flags = reinterpret_cast<int*>(base + L.flags);
    const int ta = (na + kTileR - 1) / kTileR, tb = (nb + kTileR - 1) / kTileR;
    cudaMemsetAsync(vA, 0, (size_t)ta * kTileR / 8, s);
    cudaMemsetAsync(vB, 0, (size_t)tb * kTileR / 8, s);
    const unsigned init[2] = {0x7f800000u, 0u};  // +inf, 0
    cudaMemcpyAsync(nA, init, sizeof(init), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(nB, init, sizeof(init), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(flags, 0, 16, s);
    if (ta > 0) k_match_prep<<<(ta * kTileR * 8 + 255) / 256, 256, 0, s>>>(A, na, ta, tA, vA, nA);
    if (tb > 0) k_match_prep<<<(tb * kTileR * 8 + 255) / 256, 256, 0, s>>>(B, nb, tb, tB, vB, nB);
    float* cs = reinterpret_cast<float*>(base + L.candS);
    int* cj = reinterpret_cast<int*>(base + L.candJ);
    int* bAB = reinterpret_cast<int*>(base + L.bestAB);
    int* bBA = reinterpret_cast<int*>(base + L.bestBA);
    float* d1 = reinterpret_cast<float*>(base + L.d1);
    float* d2 = reinterpret_cast<float*>(base + L.d2);
    float* d1r = reinterpret_cast<float*>(base + L.d1r);
    float* d2r = reinterpret_cast<float*>(base + L.d2r);
    if (na > 0 && nb > 0) {
        cudaError_t e = run_direction(A, na, tA, B, nb, tB, vB, nB, cs, cj, bAB, d1, d2, flags + 1, s);
        if (e != cudaSuccess) return (int)e;
        e = run_direction(B, nb, tB, A, na, tA, vA, nA, cs, cj, bBA, d1r, d2r, flags + 1, s);
        if (e != cudaSuccess) return (int)e;
        k_match_final<<<(na + 255) / 256, 256, 0, s>>>(na, bAB, d1, d2, bBA, ratio, match, dist, flags);
    } else if (na > 0) {  // nothing to match against
        k_match_none<<<(na + 255) / 256, 256, 0, s>>>(na, match, dist);
    }
    if (stats) cudaMemcpyAsync(stats, flags, 2 * sizeof(int), cudaMemcpyDeviceToDevice, s);
    return (int)cudaGetLastError();
}

}  // namespace kz
