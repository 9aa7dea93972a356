// stencil.cu — Gaussian prefilter, gradient / conductivity and the contrast factor k (sm_100a).
//
//  * prefilter: L0 = G(σ0) * I, separable tile kernel, replicate border (A6, A16).
//  * cond:      c = g(|∇(G(1) * L)|) with ∇ = Scharr step 1 (Eqs. 2-3, A5, A8); one tiled pass,
//               horizontal G1 and the horizontal Scharr taps in registers, vertical ones in shared memory.
//               Mode 0 (level 1) writes |∇|² and the image maximum of |∇| for the k histogram.
//  * khist / kfinal: 300-bin histogram of |∇| over the interior, percentile → k on the device
//               (A7), no host round trip.
#include <algorithm>
#include <cstring>

#include "kaze_internal.cuh"
#include "ptx.cuh"

namespace kz {

namespace {

constexpr float kW0c = 0.1875f, kW1c = 0.625f;  // Scharr cross smoothing (3, 10, 3)/16 (A8)
constexpr int TW = 32;  // tile width  (one warp per tile row → coalesced 128 B rows)
constexpr int TH = 32;  // tile height (block 32 x 8, four output rows per thread)


// -------------------------------------------------------------------------------------------------
// Separable Gaussian over a TW x TH output tile.  The input tile stores I(clamp(u)) for the virtual
// coordinates u of the tile + radius halo, so the separable passes equal the 2-D clamped convolution.
template <int R>
__global__ void __launch_bounds__(256) k_prefilter(const float* __restrict__ in, int64_t in_pitch,
                                                   size_t in_img_stride, float* __restrict__ out,
                                                   size_t out_img_stride, Geom g, GaussTaps t) {
    KZ_PDL_PROLOGUE();
    constexpr int LW = TW + 2 * R, LH = TH + 2 * R;
    __shared__ float tin[LH][LW];
    __shared__ float tmid[LH][TW];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const float* src = in + blockIdx.z * in_img_stride;
    const int tx = threadIdx.x, ty = threadIdx.y;
    {   // all tile loads issued before any shared store
        constexpr int KR = (LH + 7) / 8, KC = (LW + 31) / 32;
        float v[KR][KC];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int ly = ty + 8 * k;
            const float* row = src + (int64_t)clampi(y0 - R + ly, 0, g.H - 1) * in_pitch;
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int lx = tx + 32 * j;
                v[k][j] = (ly < LH && lx < LW) ? __ldg(row + clampi(x0 - R + lx, 0, g.W - 1)) : 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k)
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int ly = ty + 8 * k, lx = tx + 32 * j;
                if (ly < LH && lx < LW) tin[ly][lx] = v[k][j];
            }
    }
    float w[2 * R + 1];
#pragma unroll
    for (int d = 0; d <= 2 * R; ++d) w[d] = t.w[d];
    __syncthreads();
    for (int ly = ty; ly < LH; ly += 8) {
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(w[d], tin[ly][tx + d], acc);
        tmid[ly][tx] = acc;
    }
    __syncthreads();
    float* dst = out + blockIdx.z * out_img_stride;
    const int x = x0 + tx;
#pragma unroll
    for (int k = 0; k < TH / 8; ++k) {
        const int ly = ty + 8 * k, y = y0 + ly;
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(w[d], tmid[ly + d][tx], acc);
        if (x < g.W && y < g.H) dst[(size_t)y * g.P + x] = acc;
    }
}

// -------------------------------------------------------------------------------------------------
// Prefilter for radius 5 (σ0 = 1.6, the default) in the conductivity kernel's two-phase form: tile 64 x 56; phase 1
// one 8-column row segment per item (the 18 input columns from six 16-byte loads, all issued before the arithmetic,
// when the input rows are 16-byte aligned; clamped scalar loads otherwise) → horizontal 11-tap pass in registers
// → shared memory; phase 2 column pairs in fp32x2 (FFMA2) sliding an 11-row register window, one 8-byte store per
// row.  The 66 shared rows hold image rows clamp(y0 − 5 + r), so the vertical pass reads clamped rows exactly as
// the separable clamped convolution does.  (The generic 32x32 k_prefilter: 2.96 ms per 256-image step,
// shared-load bound at ~25 shared loads per pixel.)
constexpr int PW = 64, PH5 = 56, PR5 = 5, PRows = PH5 + 2 * PR5, PRG = 7;
__global__ void __launch_bounds__(256) k_prefilter5(const float* __restrict__ in, int64_t in_pitch,
                                                    size_t in_img_stride, float* __restrict__ out,
                                                    size_t out_img_stride, Geom g, GaussTaps t, int aligned) {
    KZ_PDL_PROLOGUE();
    __shared__ __align__(16) float sH[PRows][PW];
    const int x0 = blockIdx.x * PW, y0 = blockIdx.y * PH5, img = blockIdx.z;
    const float* src = in + img * in_img_stride;
    const int tid = threadIdx.x;
    float w[11];
#pragma unroll
    for (int d = 0; d < 11; ++d) w[d] = t.w[d];
    {
        const int sg = tid & 7, xb = x0 + 8 * sg;
        const bool fast = aligned && (xb >= 8) && (xb + 16 <= g.W);
        constexpr int NI = (PRows * 8 + 255) / 256;  // items per thread (3, the last partial)
        float v[NI][24];
#pragma unroll
        for (int it = 0; it < NI; ++it) {
            const int r = (tid >> 3) + 32 * it;
            if (r < PRows) {
                const float* row = src + (int64_t)clampi(y0 - PR5 + r, 0, g.H - 1) * in_pitch;
                if (fast) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) {
                        const float4 a = __ldg(reinterpret_cast<const float4*>(row + xb - 8) + q);
                        v[it][4 * q] = a.x;
                        v[it][4 * q + 1] = a.y;
                        v[it][4 * q + 2] = a.z;
                        v[it][4 * q + 3] = a.w;
                    }
                } else {
#pragma unroll
                    for (int q = 3; q < 21; ++q) v[it][q] = __ldg(row + clampi(xb - 8 + q, 0, g.W - 1));
                }
            }
        }
#pragma unroll
        for (int it = 0; it < NI; ++it) {
            const int r = (tid >> 3) + 32 * it;
            if (r < PRows) {
                float h[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {  // output column xb + i uses inputs xb + i − 5 .. xb + i + 5 = v[i + 3 ..]
                    float acc = w[0] * v[it][i + 3];
#pragma unroll
                    for (int d = 1; d < 11; ++d) acc = fmaf(w[d], v[it][i + 3 + d], acc);
                    h[i] = acc;
                }
                // segments 4..7 store their upper half first: conflict-free 128-bit phases (see cond_hpass)
                const int sw = sg >> 2;
                const float4 h0 = make_float4(h[0], h[1], h[2], h[3]), h1 = make_float4(h[4], h[5], h[6], h[7]);
                reinterpret_cast<float4*>(&sH[r][8 * sg])[sw] = sw ? h1 : h0;
                reinterpret_cast<float4*>(&sH[r][8 * sg])[sw ^ 1] = sw ? h0 : h1;
            }
        }
    }
    __syncthreads();
    const int cp = tid & 31, q0 = (tid >> 5) * PRG;
    const int x = x0 + 2 * cp;
    float2 wv[11];
#pragma unroll
    for (int d = 0; d < 10; ++d) wv[d] = *reinterpret_cast<const float2*>(&sH[q0 + d][2 * cp]);
    float* dst = opaque(out + img * out_img_stride);
#pragma unroll
    for (int j = 0; j < PRG; ++j) {  // output row q0 + j uses shared rows q0 + j .. q0 + j + 10
        wv[(j + 10) % 11] = *reinterpret_cast<const float2*>(&sH[q0 + j + 10][2 * cp]);
        float2 acc = __fmul2_rn(make_float2(w[0], w[0]), wv[j % 11]);
#pragma unroll
        for (int d = 1; d < 11; ++d) acc = __ffma2_rn(make_float2(w[d], w[d]), wv[(j + d) % 11], acc);
        const int y = y0 + q0 + j;
        if (y < g.H) {
            float* o = dst + (unsigned)(y * g.P + x);
            if (x + 1 < g.W) __stwb(reinterpret_cast<float2*>(o), acc);
            else if (x < g.W) __stwb(o, acc.x);
        }
    }
}

// -------------------------------------------------------------------------------------------------
// -------------------------------------------------------------------------------------------------
// |∇(G1 * L)|² → c (mode 1) or |∇|² + max|∇| (mode 0); G(σ=1) has radius 3 (A6).  Horizontal-first form: with Hl = G1_x * L (clamped columns), the Scharr step commutes
// exactly with the vertical G1 pass (they act on different axes and both clamp per axis):
//   gx = ½ Σ_dy w(dy) Va(clamp(y+dy)),  Va = G1_y * A,  A(x) = Hl(clamp(x+1)) − Hl(clamp(x−1))
//   gy = ½ [Vb(clamp(y+1)) − Vb(clamp(y−1))],  Vb = G1_y * B,  B(x) = Σ_dx w(dx) Hl(clamp(x+dx))
// with w = (3, 10, 3)/16.  Phase 1 (one 8-column row segment per item, two items per thread, all eight 16-byte
// loads issued before any arithmetic): L over 16 columns, ten Hl values, and A, B for the eight columns, stored to
// shared memory.  Phase 2 (cond_vpass_x2: a column pair × 7 rows per thread in fp32x2): vertical G1 of A and B
// sliding a 7-row register window, the vertical Scharr taps, the conductivity (or |∇|² and the interior max for the
// k histogram), and one 8-byte store per row.  Tile 64 x 56 outputs; the 64
// shared-memory rows hold image rows clamp(y0 − 4 + r), so every vertical tap reads the clamped row of its virtual
// coordinate.  The diffusivity is a template parameter and interior tiles skip every clamp and store predicate.
// (Measured on B200, 256-image 1920x1200 step: 4-column segments with per-row loads and a runtime diffusivity
// switch 30.5 ms — issue-bound at 88 instructions per pixel; the 32x32 Ls-tile kernel with three shared passes
// 39.3 ms.)
constexpr int CW2 = 64, CH2 = 56, CR2 = CH2 + 8;

// Phase-1 item: row r of the tile (image row clamp(y0 − 4 + r)), columns xb .. xb+7.
__device__ __forceinline__ void cond_load16(const float* __restrict__ row, int xb, int W, bool fast, float (&v)[16]) {
    if (fast) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(row + xb - 4) + q);
            v[4 * q] = t.x;
            v[4 * q + 1] = t.y;
            v[4 * q + 2] = t.z;
            v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldg(row + clampi(xb - 4 + q, 0, W - 1));
    }
}

__device__ __forceinline__ void cond_hpass(const float (&v)[16], const float (&w)[7], int xb, int W, bool fast, bool sw,
                                           float* __restrict__ dA, float* __restrict__ dB) {
    float h[10];  // Hl at columns xb-1 .. xb+8
#pragma unroll
    for (int q = 0; q < 10; ++q) {
        float acc = w[0] * v[q];
#pragma unroll
        for (int d = 1; d < 7; ++d) acc = fmaf(w[d], v[q + d], acc);
        h[q] = acc;
    }
    if (!fast) {  // Hl is read at clamped columns: column -1 → 0, columns >= W → W-1
        if (xb - 1 < 0) h[0] = h[1];
#pragma unroll
        for (int q = 1; q < 10; ++q)
            if (xb - 1 + q > W - 1) h[q] = h[q - 1];
    }
    float A[8], B[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        A[i] = h[i + 2] - h[i];
        B[i] = fmaf(kW0c, h[i] + h[i + 2], kW1c * h[i + 1]);
    }
    // sw: store the upper half first.  The 8 lanes of a 128-bit store phase must hit 8 distinct 4-bank groups; the
    // caller's lane mapping decides which lanes swap (a 2-way conflict on every STS.128 otherwise: 26% of the
    // kernel's shared wavefronts in the round-1 capture).
    const float4 a0 = make_float4(A[0], A[1], A[2], A[3]), a1 = make_float4(A[4], A[5], A[6], A[7]);
    const float4 b0 = make_float4(B[0], B[1], B[2], B[3]), b1 = make_float4(B[4], B[5], B[6], B[7]);
    reinterpret_cast<float4*>(dA)[sw] = sw ? a1 : a0;
    reinterpret_cast<float4*>(dB)[sw] = sw ? b1 : b0;
    reinterpret_cast<float4*>(dA)[!sw] = sw ? a0 : a1;
    reinterpret_cast<float4*>(dB)[!sw] = sw ? b0 : b1;
}

// cond_hpass for items with every tap inside the image, in packed fp32x2 (FFMA2 / FADD2 / FMUL2 on sm_100a; per
// component exactly the scalar operations in the scalar order, so the results are bit-identical): Hl pairs
// (h[2m], h[2m+1]) accumulate the aligned input pairs (v[2k], v[2k+1]) for even taps and the shifted pairs
// (v[2k+1], v[2k+2]) for odd taps; A and B pairs likewise: ~50 instead of ~102 FP instructions per item, plus the
// pair moves (staged tiles; conductivity 21.1 -> 20.9 ms per 256-image step).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ void cond_hpass_fast(const float (&v)[16], const float (&w)[7], bool sw,
                                                float* __restrict__ dA, float* __restrict__ dB) {
    float2 v2[8], vs[7];
#pragma unroll
    for (int k = 0; k < 8; ++k) v2[k] = f2(v[2 * k], v[2 * k + 1]);
#pragma unroll
    for (int k = 0; k < 7; ++k) vs[k] = f2(v[2 * k + 1], v[2 * k + 2]);
    float2 h2[5];  // (Hl at columns xb-1+2m, xb+2m)
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        float2 acc = __fmul2_rn(f2(w[0], w[0]), v2[m]);
        acc = __ffma2_rn(f2(w[1], w[1]), vs[m], acc);
        acc = __ffma2_rn(f2(w[2], w[2]), v2[m + 1], acc);
        acc = __ffma2_rn(f2(w[3], w[3]), vs[m + 1], acc);
        acc = __ffma2_rn(f2(w[4], w[4]), v2[m + 2], acc);
        acc = __ffma2_rn(f2(w[5], w[5]), vs[m + 2], acc);
        acc = __ffma2_rn(f2(w[6], w[6]), v2[m + 3], acc);
        h2[m] = acc;
    }
    float2 A2[4], B2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        A2[j] = __fadd2_rn(h2[j + 1], f2(-h2[j].x, -h2[j].y));                      // h[i+2] − h[i]
        const float2 mid = f2(h2[j].y, h2[j + 1].x);                                 // h[i+1]
        B2[j] = __ffma2_rn(f2(kW0c, kW0c), __fadd2_rn(h2[j], h2[j + 1]), __fmul2_rn(f2(kW1c, kW1c), mid));
    }
    const float4 a0 = make_float4(A2[0].x, A2[0].y, A2[1].x, A2[1].y), a1 = make_float4(A2[2].x, A2[2].y, A2[3].x, A2[3].y);
    const float4 b0 = make_float4(B2[0].x, B2[0].y, B2[1].x, B2[1].y), b1 = make_float4(B2[2].x, B2[2].y, B2[3].x, B2[3].y);
    reinterpret_cast<float4*>(dA)[sw] = sw ? a1 : a0;
    reinterpret_cast<float4*>(dB)[sw] = sw ? b1 : b0;
    reinterpret_cast<float4*>(dA)[!sw] = sw ? a0 : a1;
    reinterpret_cast<float4*>(dB)[!sw] = sw ? b0 : b1;
}

// Phase 2 of the conductivity pass in packed fp32x2 (FFMA2/FMUL2 on sm_100a): thread = (column pair cp, 7-row
// group); the vertical G1 of A and B slides down a 7-row register window of the pair's shared-memory columns (one
// 8-byte load per array and row), so each output row costs 2 loads + 14 FFMA2 + the epilogue for two pixels.
// Operation order per component is the scalar order (same rounding).
__device__ __forceinline__ float2 c2(float a) { return make_float2(a, a); }

// MODE 1 stores the conductivity; MODE 0 stores |∇|² and returns this thread's max |∇| over the image interior.
// INTERIOR (CTA-uniform, a compile-time instantiation): no clamp selects and no store predicates in the row loop.
// In MODE 1 the ½ of both central differences is folded into 1/k² as ¼ (a power-of-two scaling of every product
// and sum: bit-identical to the scaled form, two FMUL2 per row fewer).
#ifndef KZ_COND_SPLIT
#define KZ_COND_SPLIT 1
#endif
template <int MODE, int DIFF, bool INTERIOR>
__device__ __forceinline__ float cond_vpass_x2(const float (*sA)[CW2], const float (*sB)[CW2], const float (&w)[7],
                                               float* __restrict__ dst, Geom g, int x0, int y0, int tid, float ik2) {
    float lmax = 0.f;
    constexpr int RG = 7;  // output rows per thread (8 groups x 7 = CH2); 4 groups x 14 rows on half the threads
                           // (fewer window re-reads) measured 22.3 vs 21.8 ms
    const int cp = tid & 31, q0 = (tid >> 5) * RG;
    const int x = x0 + 2 * cp;
    float2 wa[7], wb[7];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        wa[d] = *reinterpret_cast<const float2*>(&sA[q0 + d][2 * cp]);
        wb[d] = *reinterpret_cast<const float2*>(&sB[q0 + d][2 * cp]);
    }
    const bool interior = INTERIOR || (KZ_COND_SPLIT == 0 && (y0 > 0) && (y0 + CH2 < g.H) && (x0 + CW2 <= g.W));
    constexpr bool kFold = MODE == 1 && KZ_COND_SPLIT;
    const float2 ik = c2(kFold ? 0.25f * ik2 : ik2);
    float2 va0 = c2(0.f), va1 = c2(0.f), vb0 = c2(0.f), vb1 = c2(0.f);  // va/vb at window rows j-2, j-1
#pragma unroll
    for (int j = 0; j < RG + 2; ++j) {  // va_j, vb_j at tile row q0 - 1 + j
        wa[(j + 6) % 7] = *reinterpret_cast<const float2*>(&sA[q0 + j + 6][2 * cp]);
        wb[(j + 6) % 7] = *reinterpret_cast<const float2*>(&sB[q0 + j + 6][2 * cp]);
        float2 a = __fmul2_rn(c2(w[0]), wa[j % 7]), b = __fmul2_rn(c2(w[0]), wb[j % 7]);
#pragma unroll
        for (int d = 1; d < 7; ++d) {
            a = __ffma2_rn(c2(w[d]), wa[(j + d) % 7], a);
            b = __ffma2_rn(c2(w[d]), wb[(j + d) % 7], b);
        }
        if (j >= 2) {  // output row r = j - 2 (tile row q0 + r): va at rows r-1, r, r+1 = va0, va1, a
            const int r = j - 2, y = y0 + q0 + r;
            float2 aup = va0, adn = a, bup = vb0, bdn = b;
            if (!interior) {
                if (y == 0) { aup = va1; bup = vb1; }
                if (y >= g.H - 1) { adn = va1; bdn = vb1; }
            }
            const float2 gx2 = __ffma2_rn(c2(kW0c), __fadd2_rn(aup, adn), __fmul2_rn(c2(kW1c), va1));
            const float2 gy2 = __fadd2_rn(bdn, make_float2(-bup.x, -bup.y));
            const float2 gx = kFold ? gx2 : __fmul2_rn(c2(0.5f), gx2);
            const float2 gy = kFold ? gy2 : __fmul2_rn(c2(0.5f), gy2);
            const float2 g2 = __ffma2_rn(gx, gx, __fmul2_rn(gy, gy));
            float2 cv;
            if constexpr (MODE == 1) {
                const float2 q = __fmul2_rn(g2, ik);
                cv = make_float2(diffusivity_g(q.x, DIFF), diffusivity_g(q.y, DIFF));
            } else {
                cv = g2;
                // the max of |∇|² and ONE square root at the end: IEEE sqrt is correctly rounded and monotonic, so
                // sqrt(max) = max(sqrt) bit for bit
                if (INTERIOR || (y >= 1 && y <= g.H - 2)) {
                    if (x >= 1 && x <= g.W - 2) lmax = fmaxf(lmax, g2.x);
                    if (x + 1 >= 1 && x + 1 <= g.W - 2) lmax = fmaxf(lmax, g2.y);
                }
            }
            float* o = dst + (unsigned)(y * g.P + x);  // dst is opaque: one IMAD.WIDE per row
            if (interior) {
                __stwb(reinterpret_cast<float2*>(o), cv);
            } else if (y < g.H) {
                if (x + 1 < g.W) __stwb(reinterpret_cast<float2*>(o), cv);
                else if (x < g.W) __stwb(o, cv.x);
            }
        }
        va0 = va1; va1 = a;
        vb0 = vb1; vb1 = b;
    }
    return MODE == 0 ? sqrtf(lmax) : lmax;
}

// Interior tiles (every tap inside the image) stage the 64 input rows x 72 columns with ONE 2-D TMA tensor copy
// (box 76 x 64: a row pitch of 76 floats puts the two rows of a 128-bit load phase 4 banks apart) instead of four
// 16-byte loads per item whose lanes use half of each 32-byte sector; border tiles keep the clamped global loads.
constexpr int kCondTP = 76;  // staged row pitch (floats)
// (Round 2, measured and dropped: persistent CTAs, 3 per SM, double-buffering the next tiles' tensor copies behind
// the current tile's work: 22.6 vs 21.1 ms per 256-image step — the 4 CTAs per SM of the per-tile form win.  Border
// tiles staged as well, their out-of-image elements replaced by the clamped values in a shared-memory fix-up pass:
// 24.8 vs 21.3 ms — the fix-up costs more than the clamped global loads it replaces.)

template <int MODE, int DIFF>
__global__ void __launch_bounds__(256) k_cond2(const __grid_constant__ CUtensorMap tmL, int use_tma,
                                               const float* __restrict__ L, size_t in_img_stride,
                                               float* __restrict__ out, size_t out_img_stride, Geom g, GaussTaps t,
                                               const float* __restrict__ kval, unsigned* __restrict__ hmax_bits) {
    KZ_PDL_PROLOGUE();
    __shared__ __align__(16) float sA[CR2][CW2];
    __shared__ __align__(16) float sB[CR2][CW2];
    __shared__ float red[8];
    extern __shared__ __align__(128) float sT[];  // [CR2][kCondTP] (TMA path only)
    __shared__ __align__(8) uint64_t bar;
    const int x0 = blockIdx.x * CW2, y0 = blockIdx.y * CH2, img = batch_image(blockIdx.z, gridDim.z, g);
    const float* src = L + img * in_img_stride;
    const int tid = threadIdx.x;
    float w[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) w[d] = t.w[d];
    const bool staged = use_tma && x0 >= 4 && x0 + CW2 + 4 <= g.W && y0 >= 4 && y0 + CH2 + 4 <= g.H;  // CTA-uniform
    if (staged) {
        if (tid == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&bar, (uint32_t)(sizeof(float) * CR2 * kCondTP));
            tma_load_3d(sT, &tmL, x0 - 4, y0 - 4, img, &bar);
        }
        // lane → (row, segment): a 128-bit phase (8 lanes) covers segments 0..3 or 4..7 of two adjacent rows, 4
        // banks apart at the 76-float pitch: conflict-free loads; odd rows store their upper half first
        const int l = tid & 31, sg = (l & 3) + 4 * ((l >> 3) & 1);
        const int r0 = 4 * (tid >> 5) + ((l >> 2) & 1) + 2 * (l >> 4);
        __syncthreads();  // the barrier is initialised before anyone waits on it
        mbar_wait(&bar, 0);
        float v0[16], v1[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 a = *reinterpret_cast<const float4*>(&sT[r0 * kCondTP + 8 * sg + 4 * q]);
            const float4 b = *reinterpret_cast<const float4*>(&sT[(r0 + 32) * kCondTP + 8 * sg + 4 * q]);
            v0[4 * q] = a.x; v0[4 * q + 1] = a.y; v0[4 * q + 2] = a.z; v0[4 * q + 3] = a.w;
            v1[4 * q] = b.x; v1[4 * q + 1] = b.y; v1[4 * q + 2] = b.z; v1[4 * q + 3] = b.w;
        }
        cond_hpass_fast(v0, w, r0 & 1, &sA[r0][8 * sg], &sB[r0][8 * sg]);
        cond_hpass_fast(v1, w, r0 & 1, &sA[r0 + 32][8 * sg], &sB[r0 + 32][8 * sg]);
    } else {
        const int sg = tid & 7, r0 = tid >> 3, xb = x0 + 8 * sg;
        const bool fast = (xb >= 4) && (xb + 12 <= g.W);
        const float* row0 = src + (size_t)clampi(y0 - 4 + r0, 0, g.H - 1) * g.P;
        const float* row1 = src + (size_t)clampi(y0 - 4 + r0 + 32, 0, g.H - 1) * g.P;
        float v0[16], v1[16];
        cond_load16(row0, xb, g.W, fast, v0);
        cond_load16(row1, xb, g.W, fast, v1);
        // the 8 lanes of a 128-bit phase are segments 0..7 of one row: halves 8sg and 8(sg + 4) share a bank group,
        // so segments 4..7 (bit 5 of xb; x0 is a multiple of 64) store their upper half first
        const bool sw = (xb >> 5) & 1;
        cond_hpass(v0, w, xb, g.W, fast, sw, &sA[r0][8 * sg], &sB[r0][8 * sg]);
        cond_hpass(v1, w, xb, g.W, fast, sw, &sA[r0 + 32][8 * sg], &sB[r0 + 32][8 * sg]);
    }
    __syncthreads();
    if constexpr (MODE == 1) {
        float* o = opaque(out + img * out_img_stride);
        const float ik2 = frcp(kval[img] * kval[img]);
        if (KZ_COND_SPLIT && (y0 > 0) && (y0 + CH2 < g.H) && (x0 + CW2 <= g.W))  // CTA-uniform
            cond_vpass_x2<1, DIFF, true>(sA, sB, w, o, g, x0, y0, tid, ik2);
        else
            cond_vpass_x2<1, DIFF, false>(sA, sB, w, o, g, x0, y0, tid, ik2);
        return;
    } else {
        float* op = opaque(out + img * out_img_stride);
        float lmax = (KZ_COND_SPLIT && (y0 > 0) && (y0 + CH2 < g.H) && (x0 + CW2 <= g.W))  // CTA-uniform
                         ? cond_vpass_x2<0, DIFF, true>(sA, sB, w, op, g, x0, y0, tid, 1.f)
                         : cond_vpass_x2<0, DIFF, false>(sA, sB, w, op, g, x0, y0, tid, 1.f);
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if ((tid & 31) == 0) red[tid >> 5] = lmax;
        __syncthreads();
        if (tid == 0) {
            float m = 0.f;
            for (int wv = 0; wv < 8; ++wv) m = fmaxf(m, red[wv]);
            atomicMax(hmax_bits + img, __float_as_uint(m));
        }
        return;
    }
}

// -------------------------------------------------------------------------------------------------
// Histogram of |∇| over the interior (A7): rows are dealt to the CTAs, each warp counts into its own shared-memory
// sub-histogram with plain shared atomics (bins <= 1024; one shared histogram above), one global add per bin.
// bin = min(floor(bins·|∇| / hmax), bins − 1) for |∇| > 0, IEEE sqrt and division (the same decision as before).
// (Measured on B200, 256-image 1920x1200 step: a flattened interior index with an integer division per pixel and
// __match_any_sync aggregation took 4.1 ms; one sub-histogram per lane index interleaved [bin][32] — conflict-free
// banks, but the same (bin, lane) counter shared by the CTA's 8 warps — 2.45 ms at 296 CTAs per image and 2.62 at
// ~37, against 1.58 for these per-warp sub-histograms.)
__global__ void __launch_bounds__(256) k_khist(const float* __restrict__ g2buf, size_t img_stride, Geom g, int bins,
                                               const unsigned* __restrict__ hmax_bits, int* __restrict__ hist) {
    KZ_PDL_PROLOGUE();
    extern __shared__ int sh[];
    const int img = blockIdx.y;
    const bool per_warp = bins <= 1024;
    const int nsub = per_warp ? 8 : 1;
    for (int i = threadIdx.x; i < bins * nsub; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int* mine = sh + (per_warp ? (threadIdx.x >> 5) * bins : 0);
    const float hmax = __uint_as_float(hmax_bits[img]);
    const float fb = (float)bins;
    const float* src = g2buf + img * img_stride;
    for (int y = 1 + blockIdx.x; y <= g.H - 2; y += gridDim.x) {
        const float* row = src + (size_t)y * g.P;
        for (int x = 1 + threadIdx.x; x <= g.W - 2; x += blockDim.x) {
            const float gm = sqrtf(__ldg(row + x));
            if (gm > 0.f) atomicAdd(mine + min((int)floorf(fb * gm / hmax), bins - 1), 1);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x) {
        int v = 0;
        for (int w = 0; w < nsub; ++w) v += sh[w * bins + i];
        if (v) atomicAdd(&hist[img * bins + i], v);
    }
}

// Percentile → k = hmax·(b+1)/bins with b the first bin whose cumulative count reaches floor(perc·n).
__global__ void k_kfinal(const int* __restrict__ hist, int bins, const unsigned* __restrict__ hmax_bits,
                         double perc, double k_override, float* __restrict__ kval, int* __restrict__ fallback) {
    KZ_PDL_PROLOGUE();
    const int img = blockIdx.x;
    if (threadIdx.x != 0) return;
    if (k_override > 0) {
        kval[img] = (float)k_override;
        fallback[img] = 0;
        return;
    }
    const int* h = hist + img * bins;
    long long n = 0;
    for (int b = 0; b < bins; ++b) n += h[b];
    if (n == 0) {
        kval[img] = 0.03f;
        fallback[img] = 1;
        return;
    }
    long long thr = (long long)floor(perc * (double)n);
    long long cum = 0;
    int b = 0;
    for (b = 0; b < bins; ++b) {
        cum += h[b];
        if (cum >= thr) break;
    }
    if (b >= bins) b = bins - 1;
    kval[img] = (float)((double)__uint_as_float(hmax_bits[img]) * (double)(b + 1) / (double)bins);
    fallback[img] = 0;
}

}  // namespace

void launch_prefilter(const float* img, int64_t in_pitch, size_t in_img_stride, float* L0, size_t out_img_stride,
                      Geom g, int nimg, const GaussTaps& t, cudaStream_t s) {
    static const int v5 = tune_knob("KAZE_PREFILTER5", 1);
    if (t.r == PR5 && v5) {
        const int aligned = ((reinterpret_cast<uintptr_t>(img) & 15) == 0) && (in_pitch % 4 == 0) && (in_img_stride % 4 == 0);
        kz_launch(k_prefilter5, dim3((g.W + PW - 1) / PW, (g.H + PH5 - 1) / PH5, nimg), dim3(256), 0, s, img, in_pitch,
                  in_img_stride, L0, out_img_stride, g, t, aligned);
        return;
    }
    dim3 grid((g.W + TW - 1) / TW, (g.H + TH - 1) / TH, nimg);
    dim3 block(32, 8);
    switch (t.r) {
#define KZ_PF(R) \
    case R: kz_launch(k_prefilter<R>, dim3(grid), dim3(block), 0, s, img, in_pitch, in_img_stride, L0, out_img_stride, g, t); break;
        KZ_PF(1) KZ_PF(2) KZ_PF(3) KZ_PF(4) KZ_PF(5) KZ_PF(6) KZ_PF(7) KZ_PF(8) KZ_PF(9) KZ_PF(10) KZ_PF(11)
        KZ_PF(12) KZ_PF(13) KZ_PF(14) KZ_PF(15) KZ_PF(16) KZ_PF(17) KZ_PF(18) KZ_PF(19) KZ_PF(20) KZ_PF(21)
        KZ_PF(22) KZ_PF(23) KZ_PF(24)
#undef KZ_PF
        default: break;
    }
}

void launch_cond(const float* L, size_t in_img_stride, float* out, size_t out_img_stride, Geom g, int nimg,
                 const GaussTaps& t1, int mode, int diffusivity, const float* kval, unsigned* hmax_bits,
                 cudaStream_t s) {
    // G(σ=1) always has radius 3 (A6), which k_cond2's 7-tap loops and 4-row halo assume
    dim3 grid((g.W + CW2 - 1) / CW2, (g.H + CH2 - 1) / CH2, nimg);
    static const int tma_knob = tune_knob("KAZE_COND_TMA", 1);
    CUtensorMap tm;
    int use_tma = 0;
    if (tma_knob) {
        const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)nimg};
        const cuuint64_t strides[2] = {(cuuint64_t)g.P * 4, (cuuint64_t)in_img_stride * 4};
        const cuuint32_t box[3] = {(cuuint32_t)kCondTP, (cuuint32_t)CR2, 1};
        use_tma = encode_f32_map(&tm, 3, L, dims, strides, box) ? 1 : 0;
    }
    if (!use_tma) memset(&tm, 0, sizeof(tm));
    const size_t smem = use_tma ? sizeof(float) * CR2 * kCondTP : 0;
    auto go = [&](auto kern) {
        if (smem) ensure_smem_optin(reinterpret_cast<const void*>(kern), (int)smem);
        kz_launch(kern, dim3(grid), dim3(256), smem, s, tm, use_tma, L, in_img_stride, out, out_img_stride, g, t1, kval,
                  hmax_bits);
    };
    if (mode == 0) {
        go(k_cond2<0, 2>);
        return;
    }
    switch (diffusivity) {
        case 1: go(k_cond2<1, 1>); break;
        case 3: go(k_cond2<1, 3>); break;
        default: go(k_cond2<1, 2>); break;
    }
}

void launch_khist(const float* g2, size_t img_stride, Geom g, int nimg, int bins, const unsigned* hmax_bits, int* hist,
                  cudaStream_t s) {
    // two CTAs per SM per image batch is plenty for a 4 B/px read (round 2: 37 / 74 / 148 / 296 CTAs per image 1.39 /
    // 1.41 / 1.44 / 1.43 ms per step — the shared-memory atomics, one per pixel, not the global merges, bound it)
    int blocks = std::min(g.H - 2, 296);
    if (blocks < 1) blocks = 1;
    const size_t smem = sizeof(int) * bins * (bins <= 1024 ? 8 : 1);
    kz_launch(k_khist, dim3(dim3(blocks, nimg)), dim3(256), smem, s, g2, img_stride, g, bins, hmax_bits, hist);
}

void launch_kfinal(const int* hist, int bins, const unsigned* hmax_bits, int nimg, double perc, double k_override,
                   float* kval, int* fallback, cudaStream_t s) {
    kz_launch(k_kfinal, dim3(nimg), dim3(32), 0, s, hist, bins, hmax_bits, perc, k_override, kval, fallback);
}


}  // namespace kz
