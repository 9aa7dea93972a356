// detect.cu — 3x3x3 extrema, edge test, 2-D sub-pixel fit and deterministic compaction (sm_100a).
//
// P:L207-214 and P:L263-281, readings A11-A13: a pixel (x, y) of level i in 1..N−2, at least one pixel from the
// border, is a keypoint iff Ldet > threshold, Ldet is strictly greater than its 26 neighbours in levels i−1, i,
// i+1, the Hessian of the response surface passes Det > 0 and Tr²/Det < (r+1)²/r (Eq. 12; Tr = Dxx + Dyy), and
// the quadratic fit offset δ = −H⁻¹∇D has |δx|, |δy| <= 1.
//
// Compaction is deterministic and ordered by (level, y, x) without a sort:
//   nms_mark : warps streaming 32-column strips down the rows — ballots produce a 1-bit-per-pixel candidate bitmap
//              and (lean kernel) per-row candidate counts by atomics; the generic kernel leaves those to k_rowcount;
//   kp_scan  : one CTA per image — exclusive scan of the row counts → row offsets, total → d_counts;
//   kp_emit  : one warp per (image, level, row) — rank of each set bit = row offset + popcounts before it; the
//              sub-pixel fit is re-evaluated (same fp32 code as the mark pass, so the same decision) and the
//              32-byte keypoint is written if its rank is below the capacity.
#include "kaze_internal.cuh"

namespace kz {

namespace {

// Edge test + sub-pixel fit on the 3x3 patch D[r][c] (r = dy+1, c = dx+1).  Returns keep.
__device__ __forceinline__ bool refine(const float (&D)[3][3], float edge_ratio, float& ox, float& oy) {
    const float cv = D[1][1];
    const float dxx = D[1][2] + D[1][0] - 2.f * cv;
    const float dyy = D[2][1] + D[0][1] - 2.f * cv;
    const float dxy = 0.25f * (D[2][2] + D[0][0] - D[0][2] - D[2][0]);
    const float gx = 0.5f * (D[1][2] - D[1][0]);
    const float gy = 0.5f * (D[2][1] - D[0][1]);
    const float det = dxx * dyy - dxy * dxy;
    if (edge_ratio > 0.f) {
        const float tr = dxx + dyy;
        if (!(det > 0.f)) return false;
        if (!(tr * tr / det < (edge_ratio + 1.f) * (edge_ratio + 1.f) / edge_ratio)) return false;
    }
    if (fabsf(det) < 1e-12f) return false;
    ox = -(dyy * gx - dxy * gy) / det;
    oy = -(dxx * gy - dxy * gx) / det;
    return fabsf(ox) <= 1.f && fabsf(oy) <= 1.f;
}

// 3-D fit in (x, y, level) on the block B[l][r][c] (l = level −1..+1), A23: the 2-D edge test on the centre slice,
// then δ = −H₃⁻¹∇D by the adjugate; keep iff |det| >= 1e-12 and |δ| <= 1 per axis.  Not inlined, so the mark and
// emit passes run the very same instructions on the same values and take the same decision.
__device__ __noinline__ bool refine3d(const float (&B)[3][3][3], float edge_ratio, float& ox, float& oy, float& os) {
    const float cv = B[1][1][1];
    const float dxx = B[1][1][2] + B[1][1][0] - 2.f * cv;
    const float dyy = B[1][2][1] + B[1][0][1] - 2.f * cv;
    const float dss = B[2][1][1] + B[0][1][1] - 2.f * cv;
    const float dxy = 0.25f * (B[1][2][2] + B[1][0][0] - B[1][0][2] - B[1][2][0]);
    const float dxs = 0.25f * (B[2][1][2] - B[2][1][0] - B[0][1][2] + B[0][1][0]);
    const float dys = 0.25f * (B[2][2][1] - B[2][0][1] - B[0][2][1] + B[0][0][1]);
    const float gx = 0.5f * (B[1][1][2] - B[1][1][0]), gy = 0.5f * (B[1][2][1] - B[1][0][1]);
    const float gs = 0.5f * (B[2][1][1] - B[0][1][1]);
    if (edge_ratio > 0.f) {
        const float det2 = dxx * dyy - dxy * dxy, tr = dxx + dyy;
        if (!(det2 > 0.f)) return false;
        if (!(tr * tr / det2 < (edge_ratio + 1.f) * (edge_ratio + 1.f) / edge_ratio)) return false;
    }
    const float a00 = dyy * dss - dys * dys, a01 = dxs * dys - dxy * dss, a02 = dxy * dys - dxs * dyy;
    const float a11 = dxx * dss - dxs * dxs, a12 = dxy * dxs - dxx * dys, a22 = dxx * dyy - dxy * dxy;
    const float det = dxx * a00 + dxy * a01 + dxs * a02;
    if (fabsf(det) < 1e-12f) return false;
    ox = -(a00 * gx + a01 * gy + a02 * gs) / det;
    oy = -(a01 * gx + a11 * gy + a12 * gs) / det;
    os = -(a02 * gx + a12 * gy + a22 * gs) / det;
    return fabsf(ox) <= 1.f && fabsf(oy) <= 1.f && fabsf(os) <= 1.f;
}

__device__ __forceinline__ bool is_keypoint(const float* __restrict__ Dm, const float* __restrict__ D0,
                                            const float* __restrict__ Dp, int P, int x, int y, float thr, float er,
                                            int use3d, float& ox, float& oy, float& os, float& v) {
    const size_t o = (size_t)y * P + x;
    v = __ldg(D0 + o);
    if (!(v > thr)) return false;
    float patch[3][3], blk[3][3][3];
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const size_t q = o + (ptrdiff_t)dy * P + dx;
            float a = __ldg(Dm + q), c = __ldg(Dp + q);
            blk[0][dy + 1][dx + 1] = a;
            blk[2][dy + 1][dx + 1] = c;
            blk[1][dy + 1][dx + 1] = __ldg(D0 + q);
            if (!(v > a) || !(v > c)) return false;
            if (dx != 0 || dy != 0) {
                float b = __ldg(D0 + q);
                if (!(v > b)) return false;
                patch[dy + 1][dx + 1] = b;
            }
        }
    patch[1][1] = v;
    blk[1][1][1] = v;
    if (use3d) return refine3d(blk, er, ox, oy, os);
    os = 0.f;
    return refine(patch, er, ox, oy);
}

// nms_mark: one WARP per (strip, NSEG-row segment, block of LB centre levels, image), streaming down the rows.
// A strip is 32 lanes over columns x0−1 .. x0+30 (x0 = 30·strip): lanes 1..30 decide columns x0 .. x0+29 and the
// edge lanes only supply neighbours, so no halo logic is needed and the bitmap word of a strip holds 30 bits
// (bit b ↔ column 30·strip + b).  The warp keeps the last three rows of its column for LB + 2 consecutive levels
// in registers, so each Ldet value is loaded once per block of LB centres (1.29 loads per pixel-level at LB = 7,
// not 3).  Per plane and row: vertical 3-max vm, two shuffles → the 3x3 max M; for a centre level also the
// 8-neighbour max N8 = max(vm_left, vm_right, up, down).  Keep iff v > thr, v > N8_i, v > M_{i−1}, v > M_{i+1}
// (strict, A11); only candidates run the edge test / sub-pixel fit.  The row loop is unrolled by three so the
// row window rotates by renaming, not by moves.
constexpr int NSEG = 63;   // rows per warp (multiple of 3).  (Streaming rows through a per-warp cp.async ring three
                           // rows ahead measured 12.3 vs 11.5 ms; a fourth register slot for the next row 19.6 vs 18.9.)
constexpr int NMS_LB = 7;  // centre levels per warp (16 levels → two blocks of 7).  Round 2, lean kernel, 256-image
                           // step: 7 centres at 4 CTAs/SM (64 registers) 11.1 ms; 6 / 5 / 4 / 3 centres at 5 / 5 / 5 / 6
                           // CTAs/SM 12.8 / 12.8 / 13.7 / 14.5; 14 centres at 2 CTAs/SM 17.5; 7 at 3 CTAs/SM 12.7.
                           // Two columns per lane (64-column warps, aligned 8-byte loads, even/odd ballots interleaved
                           // into the same bitmap; bit-identical): 19.6 / 23.7 / 26.8 ms at 4 / 5 / 7 centres..
                           // Register-ring prefetch of 1 or 2 rows ahead (window of 4/5 slots per plane): 11.1 at 4
                           // CTAs/SM (4 bytes spilled), 12.1 / 12.5 at 3, 14.2 at 2 — no gain over 11.2.
constexpr int STRIP = 30;  // output columns per strip

template <int LB, int PH, bool EXT>
__device__ __forceinline__ void nms_row(float (&w)[LB + 2][3], const float* __restrict__ base, const int (&off)[LB + 2], int P,
                                        int y, int H, int W, int x, int lane, int nc, const DetectParams& dp,
                                        uint32_t* __restrict__ bm, size_t lvl_stride, int words,
                                        const LevelTable& lt, int l0) {
    // load row y+1 (clamped) into slot (PH + 2) % 3; the window then holds rows y-1, y, y+1 in slots PH, PH+1, PH+2
    const int ro = min(y + 1, H - 1) * P;
#pragma unroll
    for (int q = 0; q < LB + 2; ++q) w[q][(PH + 2) % 3] = __ldg(base + (unsigned)(off[q] + ro));
    float M[LB + 2], N8[LB + 2];
#pragma unroll
    for (int q = 0; q < LB + 2; ++q) {
        const float up = w[q][PH % 3], ce = w[q][(PH + 1) % 3], dn = w[q][(PH + 2) % 3];
        const float vm = fmaxf(up, fmaxf(ce, dn));
        const float vl = __shfl_up_sync(0xffffffffu, vm, 1), vr = __shfl_down_sync(0xffffffffu, vm, 1);
        const float lr = fmaxf(vl, vr);
        M[q] = fmaxf(vm, lr);
        N8[q] = fmaxf(lr, fmaxf(up, dn));
    }
    const bool inside = lane >= 1 && lane <= STRIP && x >= 1 && x <= W - 2 && y >= 1 && y <= H - 2;
    if constexpr (!EXT) {
        // Default detector: per centre one FMNMX3 + FMNMX + compare + ballot; the rare candidates of every centre
        // are refined in one branch after all ballots, and lane c−1 stores centre c's bitmap word.
        uint32_t bits[LB], anyb = 0u;
#pragma unroll
        for (int c = 1; c <= LB; ++c) {
            const float v = w[c][(PH + 1) % 3];
            const float nb = fmaxf(fmaxf(N8[c], M[c - 1]), fmaxf(M[c + 1], dp.threshold));
            bits[c - 1] = c <= nc ? __ballot_sync(0xffffffffu, inside && v > nb) : 0u;
            anyb |= bits[c - 1];
        }
        if (anyb) {  // warp-uniform and rare: the level's 3x3 patch by shuffles, edge test and 2-D fit
#pragma unroll
            for (int c = 1; c <= LB; ++c) {
                if (!bits[c - 1]) continue;  // warp-uniform
                const float v = w[c][(PH + 1) % 3];
                const float u0 = w[c][PH % 3], u2 = w[c][(PH + 2) % 3];
                const float l0s = __shfl_up_sync(0xffffffffu, u0, 1), l1 = __shfl_up_sync(0xffffffffu, v, 1);
                const float l2 = __shfl_up_sync(0xffffffffu, u2, 1);
                const float r0 = __shfl_down_sync(0xffffffffu, u0, 1), r1 = __shfl_down_sync(0xffffffffu, v, 1);
                const float r2 = __shfl_down_sync(0xffffffffu, u2, 1);
                bool k = (bits[c - 1] >> lane) & 1u;
                if (k) {
                    const float patch[3][3] = {{l0s, u0, r0}, {l1, v, r1}, {l2, u2, r2}};
                    float ox, oy;
                    k = refine(patch, dp.edge_ratio, ox, oy);
                }
                bits[c - 1] = __ballot_sync(0xffffffffu, k);
            }
        }
        uint32_t mine = 0u;
#pragma unroll
        for (int c = 1; c <= LB; ++c)
            if (lane == c - 1) mine = bits[c - 1];
        if (lane < nc) bm[(size_t)lane * lvl_stride + (size_t)y * words] = (mine >> 1) & ((1u << STRIP) - 1u);
        return;
    }
#pragma unroll
    for (int c = 1; c <= LB; ++c) {
        if (c > nc) break;  // warp-uniform
        const float v = w[c][(PH + 1) % 3];
        bool k = inside && v > dp.threshold && v > N8[c] && v > M[c - 1] && v > M[c + 1];
        if (EXT && __any_sync(0xffffffffu, k)) {  // variants (A22/A23): 3x3x3 block by shuffles, window test, fit
            float blk[3][3][3];
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int rr = 0; rr < 3; ++rr) {
                    const float m = w[c - 1 + q][(PH + rr) % 3];
                    blk[q][rr][1] = m;
                    blk[q][rr][0] = __shfl_up_sync(0xffffffffu, m, 1);
                    blk[q][rr][2] = __shfl_down_sync(0xffffffffu, m, 1);
                }
            if (k && dp.exact) {  // A22: every in-image response of the (2r+1)² window at levels i±1
                const int level = l0 - 1 + c, r = max(1, lt.step[level] / 2);
                for (int q = -1; q <= 1 && k; q += 2) {
                    const float* Dq = base + off[c + q];
                    for (int dy = -r; dy <= r && k; ++dy) {
                        const int yy = y + dy;
                        if (yy < 0 || yy >= H) continue;
                        for (int dx = -r; dx <= r; ++dx) {
                            const int xx = x + dx;
                            if (xx < 0 || xx >= W) continue;
                            if (!(v > __ldg(Dq + (ptrdiff_t)yy * P + dx))) { k = false; break; }
                        }
                    }
                }
            }
            if (k) {
                float ox, oy, os;
                if (dp.refine3d) {
                    k = refine3d(blk, dp.edge_ratio, ox, oy, os);
                } else {
                    const float patch[3][3] = {{blk[1][0][0], blk[1][0][1], blk[1][0][2]},
                                               {blk[1][1][0], blk[1][1][1], blk[1][1][2]},
                                               {blk[1][2][0], blk[1][2][1], blk[1][2][2]}};
                    k = refine(patch, dp.edge_ratio, ox, oy);
                }
            }
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, k);
        if (lane == 0) bm[(size_t)(c - 1) * lvl_stride + (size_t)y * words] = (bits >> 1) & ((1u << STRIP) - 1u);
    }
}

template <int LB, bool EXT>
__global__ void __launch_bounds__(256, EXT ? 1 : 4) k_nms_mark(const float* __restrict__ Ldet, size_t img_stride, Geom g, int N,
                                                  DetectParams dp, LevelTable lt, uint32_t* __restrict__ bitmap,
                                                  int words) {
    KZ_PDL_PROLOGUE();
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (strip >= words) return;  // warp-uniform
    const int nblk = (N - 2 + LB - 1) / LB;
    const int blk = blockIdx.z % nblk, img = blockIdx.z / nblk;
    const int l0 = 1 + blk * LB;             // first centre level
    const int nc = min(LB, N - 1 - l0);      // centres in this block
    const int W = g.W, H = g.H;
    const int x = strip * STRIP - 1 + lane;
    const int xc = clampi(x, 0, W - 1);
    const int y0 = blockIdx.y * NSEG;
    const int yend = min(y0 + NSEG, H);
    // planes q = 0..LB+1 are levels l0-1+q (clamped to N-1 past the last level; never a used neighbour)
    const float* base = opaque(Ldet + img * img_stride + (size_t)(l0 - 1) * g.plane + xc);
    const int qmax = N - l0;  // last valid plane index; planes past it (short last block) re-read the last level
    int off[LB + 2];
#pragma unroll
    for (int q = 0; q < LB + 2; ++q) off[q] = min(q, qmax) * (int)g.plane;
    const size_t lvl_stride = (size_t)H * words;
    uint32_t* bm = bitmap + ((size_t)img * (N - 2) + (l0 - 1)) * lvl_stride + strip;
    float w[LB + 2][3];
    const int rm = max(y0 - 1, 0) * g.P, r0 = y0 * g.P;
#pragma unroll
    for (int q = 0; q < LB + 2; ++q) {
        w[q][0] = __ldg(base + (unsigned)(off[q] + rm));
        w[q][1] = __ldg(base + (unsigned)(off[q] + r0));
    }
    for (int y = y0; y < yend; y += 3) {
        nms_row<LB, 0, EXT>(w, base, off, g.P, y, H, W, x, lane, nc, dp, bm, lvl_stride, words, lt, l0);
        if (y + 1 < yend)
            nms_row<LB, 1, EXT>(w, base, off, g.P, y + 1, H, W, x, lane, nc, dp, bm, lvl_stride, words, lt, l0);
        if (y + 2 < yend)
            nms_row<LB, 2, EXT>(w, base, off, g.P, y + 2, H, W, x, lane, nc, dp, bm, lvl_stride, words, lt, l0);
    }
}

// Default detector, lean form: the number of centre levels NC is a compile-time constant (a launch per distinct
// block size; N = 16 gives two blocks of 7), the column part of the border test and the threshold are hoisted out
// of the row loop, and the plane offsets are uniform, so a row costs per plane one load, the vertical max, two
// shuffles and three max ops, and per centre one max3, one max, one compare and a ballot.  (The generic kernel
// above re-derived `c <= nc`, the threshold and the border predicates every row: ~30% of its instructions.)
template <int NC, int PH>
__device__ __forceinline__ void nms_row_compute(float (&w)[NC + 2][3], int y, int H, bool xin, float thr, float er,
                                                int lane, uint32_t* __restrict__ bm, size_t lvl_stride, int words,
                                                int* __restrict__ rc);

template <int NC, int PH>
__device__ __forceinline__ void nms_row_fast(float (&w)[NC + 2][3], const float* __restrict__ base,
                                             const unsigned (&off)[NC + 2], unsigned P, int y, int H, bool xin,
                                             float thr, float er, int lane, uint32_t* __restrict__ bm,
                                             size_t lvl_stride, int words, int* __restrict__ rc) {
    const unsigned ro = (unsigned)min(y + 1, H - 1) * P;
#pragma unroll
    for (int q = 0; q < NC + 2; ++q) w[q][(PH + 2) % 3] = __ldg(base + (off[q] + ro));
    // (Prefetching the row after next into L1 — prefetch.global.L1, no registers — measured 12.0 vs 10.8 ms per
    // 256-image step: the prefetches cost more issue slots and L1 tag lookups than the latency they hid.)
    nms_row_compute<NC, PH>(w, y, H, xin, thr, er, lane, bm, lvl_stride, words, rc);
}

// One row of the lean detector once row y+1 sits in window slot (PH + 2) % 3.
template <int NC, int PH>
__device__ __forceinline__ void nms_row_compute(float (&w)[NC + 2][3], int y, int H, bool xin, float thr, float er,
                                                int lane, uint32_t* __restrict__ bm, size_t lvl_stride, int words,
                                                int* __restrict__ rc) {
    float M[NC + 2], N8[NC + 2];
#pragma unroll
    for (int q = 0; q < NC + 2; ++q) {
        const float up = w[q][PH % 3], ce = w[q][(PH + 1) % 3], dn = w[q][(PH + 2) % 3];
        const float vm = fmaxf(up, fmaxf(ce, dn));
        const float vl = __shfl_up_sync(0xffffffffu, vm, 1), vr = __shfl_down_sync(0xffffffffu, vm, 1);
        M[q] = fmaxf(vm, fmaxf(vl, vr));
        if (q >= 1 && q <= NC) N8[q] = fmaxf(fmaxf(vl, vr), fmaxf(up, dn));
    }
    const bool inside = xin && y >= 1 && y <= H - 2;
    uint32_t bits[NC], anyb = 0u;
#pragma unroll
    for (int c = 1; c <= NC; ++c) {
        const float v = w[c][(PH + 1) % 3];
        const float nb = fmaxf(fmaxf(N8[c], M[c - 1]), fmaxf(M[c + 1], thr));
        bits[c - 1] = __ballot_sync(0xffffffffu, inside && v > nb);
        anyb |= bits[c - 1];
    }
    if (anyb) {  // warp-uniform and rare: the level's 3x3 patch by shuffles, edge test and 2-D fit
#pragma unroll
        for (int c = 1; c <= NC; ++c) {
            if (!bits[c - 1]) continue;  // warp-uniform
            const float v = w[c][(PH + 1) % 3];
            const float u0 = w[c][PH % 3], u2 = w[c][(PH + 2) % 3];
            const float l0s = __shfl_up_sync(0xffffffffu, u0, 1), l1 = __shfl_up_sync(0xffffffffu, v, 1);
            const float l2 = __shfl_up_sync(0xffffffffu, u2, 1);
            const float r0 = __shfl_down_sync(0xffffffffu, u0, 1), r1 = __shfl_down_sync(0xffffffffu, v, 1);
            const float r2 = __shfl_down_sync(0xffffffffu, u2, 1);
            bool k = (bits[c - 1] >> lane) & 1u;
            if (k) {
                const float patch[3][3] = {{l0s, u0, r0}, {l1, v, r1}, {l2, u2, r2}};
                float ox, oy;
                k = refine(patch, er, ox, oy);
            }
            bits[c - 1] = __ballot_sync(0xffffffffu, k);
        }
    }
    uint32_t mine = 0u;
#pragma unroll
    for (int c = 1; c <= NC; ++c)
        if (lane == c - 1) mine = bits[c - 1];
    if (lane < NC) {
        const uint32_t word = (mine >> 1) & ((1u << STRIP) - 1u);
        bm[(size_t)lane * lvl_stride + (size_t)y * words] = word;
        // the row's candidate count directly (rc: zeroed counts of this block's levels, H per level) — no separate
        // pass over the bitmap
        if (word) atomicAdd(rc + (size_t)lane * H + y, __popc(word));
    }
}

template <int NC>
__global__ void __launch_bounds__(256, 4) k_nms_mark_fast(const float* __restrict__ Ldet, size_t img_stride, Geom g,
                                                          int N, int l_first, int nblk, DetectParams dp,
                                                          uint32_t* __restrict__ bitmap, int words,
                                                          int* __restrict__ rowcnt) {
    KZ_PDL_PROLOGUE();
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (strip >= words) return;  // warp-uniform
    const int blk = blockIdx.z % nblk, img = blockIdx.z / nblk;
    const int l0 = l_first + blk * NC;  // first centre level; planes q = 0..NC+1 are levels l0−1 .. l0+NC
    const int W = g.W, H = g.H;
    const int x = strip * STRIP - 1 + lane;
    const bool xin = lane >= 1 && lane <= STRIP && x >= 1 && x <= W - 2;
    const float* base = opaque(Ldet + img * img_stride + (size_t)(l0 - 1) * g.plane + clampi(x, 0, W - 1));
    unsigned off[NC + 2];
#pragma unroll
    for (int q = 0; q < NC + 2; ++q) off[q] = (unsigned)q * (unsigned)g.plane;
    const size_t lvl_stride = (size_t)H * words;
    uint32_t* bm = bitmap + ((size_t)img * (N - 2) + (l0 - 1)) * lvl_stride + strip;
    int* rc = rowcnt + ((size_t)img * (N - 2) + (l0 - 1)) * H;
    const float thr = dp.threshold, er = dp.edge_ratio;
    const unsigned P = (unsigned)g.P;
    const int y0 = blockIdx.y * NSEG, yend = min(y0 + NSEG, H);
    float w[NC + 2][3];
    const unsigned rm = (unsigned)max(y0 - 1, 0) * P, r0 = (unsigned)y0 * P;
#pragma unroll
    for (int q = 0; q < NC + 2; ++q) {
        w[q][0] = __ldg(base + (off[q] + rm));
        w[q][1] = __ldg(base + (off[q] + r0));
    }
    for (int y = y0; y < yend; y += 3) {
        nms_row_fast<NC, 0>(w, base, off, P, y, H, xin, thr, er, lane, bm, lvl_stride, words, rc);
        if (y + 1 < yend) nms_row_fast<NC, 1>(w, base, off, P, y + 1, H, xin, thr, er, lane, bm, lvl_stride, words, rc);
        if (y + 2 < yend) nms_row_fast<NC, 2>(w, base, off, P, y + 2, H, xin, thr, er, lane, bm, lvl_stride, words, rc);
    }
}

// Row candidate counts from the bitmap: one warp per (image, level, row).
__global__ void __launch_bounds__(256) k_rowcount(const uint32_t* __restrict__ bitmap, int words, int total_rows,
                                                  int* __restrict__ rowcnt) {
    KZ_PDL_PROLOGUE();
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= total_rows) return;
    const uint32_t* bm = bitmap + (size_t)q * words;
    int c = 0;
    for (int w = lane; w < words; w += 32) c += __popc(bm[w]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) rowcnt[q] = c;
}

// One CTA per image: exclusive scan of R row counts.
__global__ void __launch_bounds__(1024) k_kp_scan(const int* __restrict__ rowcnt, int R, int* __restrict__ rowoff,
                                                  int* __restrict__ counts) {
    KZ_PDL_PROLOGUE();
    __shared__ int wsum[32];
    const int img = blockIdx.x;
    const int* rc = rowcnt + (size_t)img * R;
    int* ro = rowoff + (size_t)img * R;
    const int per = (R + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(b + per, R);
    int local = 0;
    for (int i = b; i < e; ++i) local += rc[i];
    // block exclusive scan of `local`
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        wsum[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    int run = incl - local + (warp > 0 ? wsum[warp - 1] : 0);
    for (int i = b; i < e; ++i) {
        ro[i] = run;
        run += rc[i];
    }
    if (threadIdx.x == blockDim.x - 1) counts[img] = run;
}

// One WARP per (image, level, row); 8 rows per CTA.  (Four rows per warp, their counts and offsets in one load each:
// 3.2 vs 2.8 ms per 256-image step — the rows then run serially in the warp.)  Lane w of a 32-word step owns bitmap word w: an inclusive warp
// scan of the word popcounts gives each word's rank base, and the lane walks its set bits in x order.
__global__ void __launch_bounds__(256) k_kp_emit(const float* __restrict__ Ldet, size_t img_stride, Geom g,
                                                 LevelTable lt, DetectParams dp, const uint32_t* __restrict__ bitmap,
                                                 const int* __restrict__ rowcnt, const int* __restrict__ rowoff,
                                                 kaze_keypoint* __restrict__ kps, int total_rows) {
    KZ_PDL_PROLOGUE();
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5);  // flat row id over (img, level-1, y)
    if (q >= total_rows) return;
    if (rowcnt[q] == 0) return;  // warp-uniform
    const int N = lt.n;
    const int y = q % g.H, rest = q / g.H, li = rest % (N - 2), img = rest / (N - 2), level = li + 1;
    const int words = (g.W + STRIP - 1) / STRIP;
    const uint32_t* bm = bitmap + (size_t)q * words;
    const float* D0 = Ldet + img * img_stride + (size_t)level * g.plane;
    int run = rowoff[q];
    for (int w0 = 0; w0 < words; w0 += 32) {
        uint32_t word = (w0 + lane < words) ? bm[w0 + lane] : 0u;
        const int c = __popc(word);
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        int rank = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
        while (word) {
            const int bit = __ffs(word) - 1;
            word &= word - 1;
            if (rank < dp.cap) {
                const int x = (w0 + lane) * STRIP + bit;
                float ox = 0.f, oy = 0.f, os = 0.f, v = 0.f;
                if (dp.refine3d) {
                    is_keypoint(D0 - g.plane, D0, D0 + g.plane, g.P, x, y, dp.threshold, dp.edge_ratio, 1, ox, oy,
                                os, v);
                } else {
                    // the mark pass has decided; the 2-D fit needs only the level's 3x3 patch — the very values and
                    // code of the mark pass, so the very offsets (9 loads instead of the 26-neighbour re-check's 35)
                    const size_t o = (size_t)y * g.P + x;
                    float patch[3][3];
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                        for (int dx = -1; dx <= 1; ++dx) patch[dy + 1][dx + 1] = __ldg(D0 + o + (ptrdiff_t)dy * g.P + dx);
                    v = patch[1][1];
                    refine(patch, dp.edge_ratio, ox, oy);
                }
                kaze_keypoint kp;
                kp.x = (float)x + ox;
                kp.y = (float)y + oy;
                kp.sigma = dp.refine3d ? lt.sigma[level] * exp2f(os / (float)lt.S) : lt.sigma[level];
                kp.response = v;
                kp.angle = 0.f;
                kp.level = level;
                kp.octave = (int16_t)(level / lt.S);
                kp.sublevel = (int16_t)(level % lt.S);
                kp.flags = 0;
                kps[(size_t)img * dp.cap + rank] = kp;
            }
            ++rank;
        }
    }
}

}  // namespace

int nms_words(int W) { return (W + STRIP - 1) / STRIP; }

int launch_nms_mark(const float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt, DetectParams dp,
                    uint32_t* bitmap, int* rowcnt, cudaStream_t s) {
    int nk = 1;  // kernels launched (the generic paths add k_rowcount)
    const int N = lt.n;
    const int words = nms_words(g.W);
    const int nblk = (N - 2 + NMS_LB - 1) / NMS_LB;
    dim3 grid((words + 7) / 8, (g.H + NSEG - 1) / NSEG, nimg * nblk);
    static const int lean = tune_knob("KAZE_NMS_LEAN", 1);
    if (dp.exact || dp.refine3d) {  // detector variants (§8 f2) in their own instantiation: the default stays lean
        kz_launch(k_nms_mark<NMS_LB, true>, dim3(grid), dim3(256), 0, s, Ldet, img_stride, g, N, dp, lt, bitmap, words);
    } else if (!lean) {
        kz_launch(k_nms_mark<NMS_LB, false>, dim3(grid), dim3(256), 0, s, Ldet, img_stride, g, N, dp, lt, bitmap, words);
    } else {
        // full blocks of NMS_LB centre levels in one launch, the remainder (if any) in a second
        const int full = (N - 2) / NMS_LB, rem = (N - 2) - full * NMS_LB;
        nk += (full > 0) + (rem > 0) - 1;
        // (A variant streaming the rows through a 6-slot shared-memory ring filled by 1-D bulk copies, 5 rows
        // ahead of the warps, measured 14.9 vs 11.5 ms per 256-image step: the mbarrier waits and the extra
        // bookkeeping cost more issue slots than the hidden load latency saved.)
        cudaMemsetAsync(rowcnt, 0, sizeof(int) * (size_t)g.H * (N - 2) * nimg, s);  // counted by the mark pass
        if (full > 0)
            kz_launch(k_nms_mark_fast<NMS_LB>, dim3(dim3(grid.x, grid.y, nimg * full)), dim3(256), 0, s, Ldet,
                      img_stride, g, N, 1, full, dp, bitmap, words, rowcnt);
        const int lr = 1 + full * NMS_LB;
        switch (rem) {
#define KZ_NMS_REM(R)                                                                                              \
    case R:                                                                                                        \
        kz_launch(k_nms_mark_fast<R>, dim3(dim3(grid.x, grid.y, nimg)), dim3(256), 0, s, Ldet, img_stride, g, N, lr, \
                  1, dp, bitmap, words, rowcnt);                                                                   \
        break;
            KZ_NMS_REM(1) KZ_NMS_REM(2) KZ_NMS_REM(3) KZ_NMS_REM(4) KZ_NMS_REM(5) KZ_NMS_REM(6)
#undef KZ_NMS_REM
            default: break;
        }
        return nk;  // the lean mark pass counted the rows itself (0.7 ms per 256-image step of k_rowcount saved)
    }
    const int total = g.H * (N - 2) * nimg;
    kz_launch(k_rowcount, dim3((total + 7) / 8), dim3(256), 0, s, bitmap, words, total, rowcnt);
    return nk + 1;
}

void launch_kp_scan(const int* rowcnt, int rows_per_img, int nimg, int* rowoff, int* counts, cudaStream_t s) {
    kz_launch(k_kp_scan, dim3(nimg), dim3(1024), 0, s, rowcnt, rows_per_img, rowoff, counts);
}

void launch_kp_emit(const float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt, DetectParams dp,
                    const uint32_t* bitmap, const int* rowcnt, const int* rowoff, kaze_keypoint* kps, cudaStream_t s) {
    const int total = g.H * (lt.n - 2) * nimg;
    kz_launch(k_kp_emit, dim3((total + 7) / 8), dim3(256), 0, s, Ldet, img_stride, g, lt, dp, bitmap, rowcnt, rowoff, kps, total);
}

}  // namespace kz
