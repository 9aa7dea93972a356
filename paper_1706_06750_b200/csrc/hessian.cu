// hessian.cu — multiscale derivatives and the scale-normalised Hessian determinant (Eq. 8; A9, A10).
//
// With the dilated Scharr operator at step s (taps at 0, ±s; derivative (−1, 0, 1)/2 after the s-normalisation,
// cross smoothing (3, 10, 3)/16) written N_x, N_y:
//     Lx = N_x L,  Ly = N_y L,  Ldet = N_x(Lx)·N_y(Ly) − N_y(Lx)²
// which equals s⁴(LxxLyy − Lxy²) with per-pixel derivatives (the factor s per derivative order is absorbed in
// N).  Second derivatives read the MATERIALISED first derivatives at clamped coordinates (A10), so they are two
// passes in principle: hess_first (L → Lx, Ly) and hess_det (Lx, Ly → Ldet).  The default is ONE fused pass
// (k_hess_fused, 16 instead of 24 B/px): a CTA owns one chain of rows y0 + j·s and a block of columns, keeps the
// chain's (Lx, Ly) with an s-column halo in shared memory and forms Ldet from it (256-image 1920x1200 step: 39.8
// vs 45.8 ms for the two chain passes).  One launch covers every level of every image (blockIdx.z packs (image,
// level)); the per-level step s_i comes from the LevelTable.  (An earlier fused form on square tiles recomputed a
// (T+4s)² halo and lost to the two passes: 80-87 µs vs 59 µs per level and 4 images.)
#include "kaze_internal.cuh"

namespace kz {

namespace {

// The Scharr step-s operators in separable form (A8, A9): with the row terms
//   D(r) = L(r, x+s) − L(r, x−s)      (x-difference)      Mh(r) = hw0·(L(r, x−s) + L(r, x+s)) + hw1·L(r, x)   (x-smoothing)
// and hw = (3, 10, 3)/32 (the (3, 10, 3)/16 cross smoothing with the ½ of the central difference folded in — a
// power-of-two scaling, so exact), N_x L = hw0·(D(y−s) + D(y+s)) + hw1·D(y) and N_y L = Mh(y+s) − Mh(y−s).  Every
// row term is computed once and shared by the up-to-three outputs that use it (the chain rows of phase A, the
// ring rows of phase B): 4 instead of 7 operations per derivative.  All paths (fused fast / clamped, two-pass)
// use exactly these operations, so a value computed by two CTAs (column halos) is bit-identical.
constexpr float hw0 = 0.09375f, hw1 = 0.3125f;  // (3, 10, 3) / 32

struct RowTerms {  // D, Mh of one row of taps (x−s, x, x+s)
    float d, mh;
};
__device__ __forceinline__ RowTerms row_terms(float a, float m, float c) { return {c - a, fmaf(hw0, a + c, hw1 * m)}; }
// (N_x L, N_y L) at the middle row from the row terms of rows y−s, y, y+s
__device__ __forceinline__ float2 first_from_rows(RowTerms r0, RowTerms r1, RowTerms r2) {
    return make_float2(fmaf(hw0, r0.d + r2.d, hw1 * r1.d), r2.mh - r0.mh);
}
// Second-stage row terms of one ring row (columns x−s, x, x+s of (Lx, Ly)): E = x-difference of Lx, P / Q =
// x-smoothing of Lx / Ly; then N_x(Lx) = hw0·(E0 + E2) + hw1·E1, N_y(Lx) = P2 − P0, N_y(Ly) = Q2 − Q0.
// P and Q are the same operations on the two components, so they run as one packed fp32x2 op each (FADD2 / FMUL2 /
// FFMA2 on sm_100a: per component exactly the scalar operation, same rounding): 4 instead of 7 instructions per ring
// row, and the N_y differences as one FADD2 (fused Hessian 33.9 -> 33.3 ms per 256-image step).
struct RingTerms {
    float e;
    float2 pq;
};
__device__ __forceinline__ RingTerms ring_terms(float2 a, float2 b, float2 c) {
    return {c.x - a.x, __ffma2_rn(make_float2(hw0, hw0), __fadd2_rn(a, c), __fmul2_rn(make_float2(hw1, hw1), b))};
}
__device__ __forceinline__ float det_from_terms(RingTerms r0, RingTerms r1, RingTerms r2) {
    const float lxx = fmaf(hw0, r0.e + r2.e, hw1 * r1.e);                     // N_x(Lx)
    const float2 d = __fadd2_rn(r2.pq, make_float2(-r0.pq.x, -r0.pq.y));      // (N_y(Lx), N_y(Ly))
    return lxx * d.y - d.x * d.x;
}
__device__ __forceinline__ float det_from_ring(float2 a, float2 b, float2 c, float2 d, float2 e, float2 f, float2 h,
                                               float2 i, float2 j) {
    return det_from_terms(ring_terms(a, b, c), ring_terms(d, e, f), ring_terms(h, i, j));
}

// Chain form: a thread computes R outputs of one column at rows y_j = y_0 + j·s (j < R) — a "chain" in the row
// residue class of y_0 mod s.  Output j reads rows y_j − s, y_j, y_j + s = chain rows j−1, j, j+1, so the R outputs
// need (R + 2) rows × 3 taps instead of 8R taps: 44% fewer L1 wavefronts at R = 4, 61% at R = 8.  Chains tile the
// rows band by band: band b = [b·R·s, (b+1)·R·s) holds the s chains y_0 = b·R·s + r, r < s.  Every tap is read at
// clamped coordinates (A10/A16); the clamp of row y_j ± s equals the clamp of the neighbouring chain row.
constexpr int kChainR = 8;  // measured at 1920x1200 (256-image step): R = 8 51.3 ms, 12 53.0, 4 61.1, 32x32 tiles 59.2

// Chains of one level: s per band, ceil(H / (R·s)) bands.  grid.y covers the largest level; blocks past a level's
// chain count exit at once.  b = ch / s via a float quotient: (ch + ½)/s stays >= 1/(2s) away from an integer, far
// beyond the error of __fdividef at these sizes (ch < 2^16, s < 64).
__device__ __forceinline__ int chain_band(int ch, int s) { return (int)__fdividef((float)ch + 0.5f, (float)s); }

// Interior chains (every tap row and column inside the image — all but the border warps) take a clamp-free path
// with the step s as a compile-time constant: one row pointer per chain row and the x − s, x, x + s taps as
// immediate offsets from it (~4 instructions per 3 loads instead of ~10).  Border chains and steps above
// kMaxTemplStep use the clamped generic path.  (The two-pass chain kernels dispatch on s per CTA; s is uniform per
// level.  The fused kernel below keeps s in a register instead: its two phases are long enough that the code size
// of 24 unrolled cases cost more than the immediate offsets save.)
constexpr int kMaxTemplStep = 24;

template <int R, int SC, class T>
__device__ __forceinline__ bool chain_setup(Geom g, int s_rt, int ch, int x, int& s, int& y0, bool& fast) {
    s = SC > 0 ? SC : s_rt;
    const int nch = s * ((g.H + R * s - 1) / (R * s));
    if (ch >= nch || x >= g.W) return false;
    const int b = SC > 0 ? ch / SC : chain_band(ch, s);
    y0 = b * R * s + (ch - b * s);
    fast = SC > 0 && y0 >= s && y0 + R * s <= g.H - 1 && x >= s && x + s <= g.W - 1;
    return true;
}

// Loads columns x−s, x, x+s of chain rows −1..R (rows y0 + (k−1)s, clamped on the generic path).
template <int R, int SC, class T>
__device__ __forceinline__ void chain_load(const T* __restrict__ src, Geom g, int s, int y0, int x, bool fast,
                                           T (&a)[R + 2], T (&m)[R + 2], T (&c)[R + 2]) {
    if (SC > 0 && fast) {
#pragma unroll
        for (int k = 0; k < R + 2; ++k) {
            const T* p = src + (unsigned)((y0 + (k - 1) * SC) * g.P + x);
            a[k] = __ldg(p - SC);
            m[k] = __ldg(p);
            c[k] = __ldg(p + SC);
        }
    } else {
        const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
#pragma unroll
        for (int k = 0; k < R + 2; ++k) {
            const int ro = clampi(y0 + (k - 1) * s, 0, g.H - 1) * g.P;
            a[k] = __ldg(src + (unsigned)(ro + xm));  // unsigned 32-bit offsets: one IMAD.WIDE.U32 per address
            m[k] = __ldg(src + (unsigned)(ro + x));
            c[k] = __ldg(src + (unsigned)(ro + xp));
        }
    }
}

template <int R, int SC>
__device__ __forceinline__ void hess_first_body(const float* __restrict__ L, float2* __restrict__ D, Geom g, int s_rt,
                                                int ch, int x) {
    int s, y0;
    bool fast;
    if (!chain_setup<R, SC, float>(g, s_rt, ch, x, s, y0, fast)) return;
    float a[R + 2], m[R + 2], c[R + 2];  // columns x−s, x, x+s of chain rows −1..R
    chain_load<R, SC, float>(L, g, s, y0, x, fast, a, m, c);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int y = y0 + j * s;
        const float2 v = first_from_rows(row_terms(a[j], m[j], c[j]), row_terms(a[j + 1], m[j + 1], c[j + 1]),
                                         row_terms(a[j + 2], m[j + 2], c[j + 2]));
        if (fast || y < g.H) __stwb(D + (unsigned)(y * g.P + x), v);
    }
}

template <int R, int SC>
__device__ __forceinline__ void hess_det_body(const float2* __restrict__ D, float* __restrict__ O, Geom g, int s_rt,
                                              int ch, int x) {
    int s, y0;
    bool fast;
    if (!chain_setup<R, SC, float2>(g, s_rt, ch, x, s, y0, fast)) return;
    float2 a[R + 2], m[R + 2], c[R + 2];
    chain_load<R, SC, float2>(D, g, s, y0, x, fast, a, m, c);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int y = y0 + j * s;
        const float v = det_from_ring(a[j], m[j], c[j], a[j + 1], m[j + 1], c[j + 1], a[j + 2], m[j + 2], c[j + 2]);
        if (fast || y < g.H) __stwb(O + (unsigned)(y * g.P + x), v);
    }
}

#define KZ_STEP_CASES(F) \
    F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14) F(15) F(16) F(17) F(18) F(19) F(20) \
    F(21) F(22) F(23) F(24)

template <int R>
__global__ void __launch_bounds__(256) k_hess_first_chain(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                          size_t img_stride, Geom g, LevelTable lt) {
    KZ_PDL_PROLOGUE();
    const int img = chain_band(blockIdx.z, lt.n), level = blockIdx.z - img * lt.n;
    const int s = lt.step[level];
    const int ch = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const size_t base = img * img_stride + (size_t)level * g.plane;
    const float* L = opaque(Lt + base);
    float2* D = opaque(Lxy + base);
    switch (s) {
#define KZ_CASE(S) \
    case S: hess_first_body<R, S>(L, D, g, s, ch, x); break;
        KZ_STEP_CASES(KZ_CASE)
#undef KZ_CASE
        default: hess_first_body<R, 0>(L, D, g, s, ch, x); break;
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_hess_det_chain(const float2* __restrict__ Lxy, float* __restrict__ Ldet,
                                                        size_t img_stride, Geom g, LevelTable lt) {
    KZ_PDL_PROLOGUE();
    const int img = chain_band(blockIdx.z, lt.n), level = blockIdx.z - img * lt.n;
    const int s = lt.step[level];
    const int ch = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const size_t base = img * img_stride + (size_t)level * g.plane;
    const float2* D = opaque(Lxy + base);
    float* O = opaque(Ldet + base);
    switch (s) {
#define KZ_CASE(S) \
    case S: hess_det_body<R, S>(D, O, g, s, ch, x); break;
        KZ_STEP_CASES(KZ_CASE)
#undef KZ_CASE
        default: hess_det_body<R, 0>(D, O, g, s, ch, x); break;
    }
}

// ---------------------------------------------------------------------------------------------------------------
// Fused form (one pass, 16 instead of 24 B/px): a CTA owns ONE chain (rows y0 + j·s, j < R, of one residue class)
// and CW output columns [x0, x0 + CW).  Phase A: thread t computes (Lx, Ly) of virtual column x0 − s + t at the
// chain rows −1..R — at clamped coordinates, exactly what the second pass of the two-pass form reads (A10) — into
// shared memory, and stores the rows 0..R−1 of the output columns to the Lxy pyramid (the descriptor samples it).
// Phase B: thread t < CW forms Ldet of column x0 + t from the ring at columns ±s, rows ±1 in shared memory.  Only
// the s-column halo of (Lx, Ly) is recomputed (CW + 2s ≤ 256 columns per 256 threads), and the L taps of the
// column halo and of the two extra chain rows come from L1/L2.  Same arithmetic, same order as the two passes:
// bit-identical results.
#ifndef KZ_HESS_R
#define KZ_HESS_R 12
#endif
#ifndef KZ_HESS_MINB
#define KZ_HESS_MINB 6
#endif
constexpr int kFusedR = KZ_HESS_R;  // measured (256-image step): R = 16 38.3 ms, 8 39.8, 4 43.4, 20 44.1, 32 77.5 (round 2,
                                    // with the row-term form: 16 36.9, 12 38.5 (32 registers, 7 CTAs/SM), 20 41.5;
                                    // 512-thread CTAs (CW = 480/448) 46.4 vs 38.7).  With the one-path kernel (step in
                                    // a register): R = 12 at 6 CTAs/SM 33.0 vs 33.6 at 16, 33.3 at 12 with 7 CTAs/SM,
                                    // 33.5 at 16 with 5, 33.3 at 20 with 5.  Session 3 (one box): R = 12 33.65 vs
                                    // R = 14 at 6 (spills) 34.67, R = 10 at 7 CTAs/SM (32 registers) 34.0.
// (Round 2, measured and dropped: border chains are 35% of the CTAs at 1920x1200 and cost ~1.7x an interior chain
// (all chains forced onto the border path: 43.8 vs 31.8 ms at equal clocks), but hoisting their 3(R + 4) loads like
// the interior path — one clamped path for every chain 39.4, clamped hoisting for the border chains only 35.2, for
// the row-border chains only 34.5, vs 33.1 ms — spills at the 40-register budget of 6 CTAs per SM.)
// (Round 2, measured and dropped: a compact grid (blockIdx.x = work item of the image in (level, chain, column block)
// order, decoded from a per-level table) instead of the (columns, chains, image x level) grid sized by the largest
// level, whose 21% empty CTAs exit at once: 35.3 vs 33.4 ms — the decode costs more than the empty CTAs.)
// (Round 2, measured and dropped: the (Lx, Ly) rows leaving through 1-D TMA bulk stores straight from the shared rows
// (columns shifted by s & 1 for 16-byte alignment) instead of per-thread 8-byte stores: 33.9/34.1 vs 34.2/34.1 ms —
// no change beyond noise, and the extra state spills at 40 registers.)
// (Round 2, measured and dropped: phase A as a rolling window of three tap rows with bounded unrolling, to cut the
// ~1600 straight-line instructions per step case (ncu: 16% of stalls are "no instruction"): unroll 1/2/4/8/full
// 46.1/38.4/38.6/34.6/35.7 vs 34.0 ms — hoisting all tap loads ahead of the arithmetic matters more.)
// (Round 2, measured and dropped: the chain's L tap rows staged by ONE TMA tensor copy per CTA through a per-level
// 4-D "chain view" map (x: W, r: s, q: ⌈H/s⌉, image; byte strides 4, 4P, 4sP, image stride), box (256, 1, R + 4, 1)
// at (x0 − 2s, r, b·R − 2, img), phase A reading its taps from shared memory — bit-identical results, but the
// (R + 4) KB tile on top of the (Lx, Ly) rows costs occupancy and the copy latency is exposed per CTA: R = 16/14/12
// at 3/4/5 CTAs per SM 43.9/38.0/36.1 vs 34.1 ms per 256-image step; persistent CTAs double-buffering the next
// items' copies R = 12/8/16 at 3/4/2 CTAs per SM 41.8/64.5/47.9 vs 34.4.  The kernel needs its 48 warps per SM.  Also
// measured: a 4-D tiled copy whose first coordinate is not a multiple of 4 floats faults with an illegal
// instruction on B200, a 3-D one does not.)

// CW + 2s <= 256.  (Phase-A threads on 32-float aligned columns x0 − 32 + t with CW = 192 for every s — aligned centre
// taps, more halo blocks — measured 44.8 vs 38.6 ms.)
__device__ __forceinline__ int fused_cw(int s) { return s <= 16 ? 224 : 192; }
__host__ inline int fused_cw_host(int s) { return s <= 16 ? 224 : 192; }

template <int R>
__device__ __forceinline__ void hess_fused_body(const float* __restrict__ L, float2* __restrict__ D, float* __restrict__ O,
                                                Geom g, int s, int ch, int xb, float2 (*sm)[256], bool keep_d) {
    const int cw = fused_cw(s);
    const int nch = s * ((g.H + R * s - 1) / (R * s));
    const int x0 = xb * cw;
    if (ch >= nch || x0 >= g.W) return;  // CTA-uniform
    const int b = chain_band(ch, s);
    const int y0 = b * R * s + (ch - b * s);
    const int t = threadIdx.x;
    const int vc = x0 - s + t;  // virtual column of this thread in phase A
    const bool in_a = t < cw + 2 * s;
    const bool fast = y0 >= 2 * s && y0 + (R + 1) * s <= g.H - 1 && x0 >= 2 * s && x0 + cw + 2 * s <= g.W;
    if (in_a) {
        const int cc = clampi(vc, 0, g.W - 1);
        const bool store_col = keep_d && vc >= x0 && vc < x0 + cw && vc < g.W;
        if (fast) {
            // chain rows k = -2..R+1 of columns cc - s, cc, cc + s (no clamps anywhere); each row's terms once
            RowTerms rt[R + 4];
#pragma unroll
            for (int k = 0; k < R + 4; ++k) {
                const float* p = L + (unsigned)((y0 + (k - 2) * s) * g.P + cc);
                rt[k] = row_terms(__ldg(p - s), __ldg(p), __ldg(p + s));
            }
#pragma unroll
            for (int k = 0; k < R + 2; ++k) {  // chain row k - 1 uses rows k, k+1, k+2 of the arrays
                const float2 v = first_from_rows(rt[k], rt[k + 1], rt[k + 2]);
                sm[k][t] = v;
                if (k >= 1 && k <= R && store_col) __stwb(D + (unsigned)((y0 + (k - 1) * s) * g.P + vc), v);
            }
        } else {
            // Border chains (and steps without a template case): the same sliding row terms, over CLAMPED rows and
            // columns.  For a chain row yv inside the image its taps are rows clamp(yv − s), yv, clamp(yv + s) —
            // exactly rows k, k+1, k+2 of the clamped array.  A chain row outside the image holds (Lx, Ly) of the
            // clamped image row (A10: the second derivatives read the first ones at clamped coordinates), i.e. of
            // row 0 (taps 0, 0, s) or row H−1 (taps H−1−s, H−1, H−1), computed once when the chain needs it.  Same
            // operations on the same values as the per-row form this replaces (bit-identical), ~1/3 of its loads
            // (R + 4 tap rows instead of 3(R + 2)).
            const int xm = max(cc - s, 0), xp = min(cc + s, g.W - 1);
            auto terms_at = [&](int y) {
                const unsigned ro = (unsigned)(clampi(y, 0, g.H - 1) * g.P);
                return row_terms(__ldg(L + (ro + xm)), __ldg(L + (ro + cc)), __ldg(L + (ro + xp)));
            };
            float2 top = make_float2(0.f, 0.f), bot = top;
            if (y0 - s < 0) {  // chain row −1 (and only it, y0 < s) lies above the image
                const RowTerms r0 = terms_at(0);
                top = first_from_rows(r0, r0, terms_at(s));
            }
            if (y0 + R * s > g.H - 1) {  // some chain rows lie below the image
                const RowTerms rl = terms_at(g.H - 1);
                bot = first_from_rows(terms_at(g.H - 1 - s), rl, rl);
            }
            RowTerms ra = terms_at(y0 - 2 * s), rb = terms_at(y0 - s);  // a rolling window of three tap rows
#pragma unroll
            for (int k = 0; k < R + 2; ++k) {
                const RowTerms rc = terms_at(y0 + k * s);
                const int yv = y0 + (k - 1) * s;  // chain row k - 1 (virtual)
                const float2 v = yv < 0 ? top : (yv > g.H - 1 ? bot : first_from_rows(ra, rb, rc));
                sm[k][t] = v;
                if (k >= 1 && k <= R && store_col && yv < g.H) __stwb(D + (unsigned)(yv * g.P + vc), v);
                ra = rb;
                rb = rc;
            }
        }
    }
    __syncthreads();
    if (t < cw && x0 + t < g.W) {
        // ring: columns x − s, x, x + s ↔ shared columns t, t + s, t + 2s; chain rows −1..R ↔ shared rows 0..R+1;
        // each ring row's terms (E, P, Q) once, shared by the three outputs that read the row
        RingTerms r0 = ring_terms(sm[0][t], sm[0][t + s], sm[0][t + 2 * s]);
        RingTerms r1 = ring_terms(sm[1][t], sm[1][t + s], sm[1][t + 2 * s]);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int y = y0 + j * s;
            if (!fast && y >= g.H) break;
            const RingTerms r2 = ring_terms(sm[j + 2][t], sm[j + 2][t + s], sm[j + 2][t + 2 * s]);
            __stwb(O + (unsigned)(y * g.P + x0 + t), det_from_terms(r0, r1, r2));
            r0 = r1;
            r1 = r2;
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256, KZ_HESS_MINB) k_hess_fused(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                    float* __restrict__ Ldet, size_t img_stride, Geom g, LevelTable lt,
                                                    int keep_edges) {
    KZ_PDL_PROLOGUE();
    __shared__ float2 sm[R + 2][256];  // 28 KB at R = 12.  (Staging the L taps in shared memory as well — each
                                       // loaded once instead of three times through L1 — measured slower: 76.7 ms.)
    const int img = chain_band(blockIdx.z, lt.n), level = blockIdx.z - img * lt.n;
    const int s = lt.step[level];
    const size_t base = img * img_stride + (size_t)level * g.plane;
    const float* L = opaque(Lt + base);
    float2* D = opaque(Lxy + base);
    float* O = opaque(Ldet + base);
    // (Lx, Ly) of the first and last level only feed their own Ldet (no keypoints there): not stored by default
    const bool keep_d = keep_edges || (level > 0 && level < lt.n - 1);
    // One code path for every step: s stays in a register.  (A switch over compile-time steps 1..24 with the x ± s
    // taps as immediate offsets produced 24 cases of ~1600 straight-line instructions — 38k instructions, 16% of the
    // stalls "no instruction" — and measured 33.2 vs 33.0 ms per 256-image step for this 1.9k-instruction form.)
    hess_fused_body<R>(L, D, O, g, s, blockIdx.y, blockIdx.x, sm, keep_d);
}

template <int R>
int max_chain_blocks(Geom g, const LevelTable& lt) {
    int m = 1;
    for (int l = 0; l < lt.n; ++l) {
        const int s = lt.step[l];
        m = max(m, (s * ((g.H + R * s - 1) / (R * s)) + 7) / 8);
    }
    return m;
}

__global__ void k_component_copy(float2* __restrict__ plane, int comp, float* __restrict__ tight, int to_tight,
                                 Geom g) {
    KZ_PDL_PROLOGUE();
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= g.W) return;
    float* e = reinterpret_cast<float*>(plane + (size_t)y * g.P + x) + comp;
    if (to_tight) tight[(size_t)y * g.W + x] = *e;
    else *e = tight[(size_t)y * g.W + x];
}

}  // namespace

void launch_hess_first(const float* Lt, float2* Lxy, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                       cudaStream_t s) {
    const dim3 grid((g.W + 31) / 32, max_chain_blocks<kChainR>(g, lt), nimg * lt.n);
    kz_launch(k_hess_first_chain<kChainR>, dim3(grid), dim3(dim3(32, 8)), 0, s, Lt, Lxy, img_stride, g, lt);
}

void launch_hess_det(const float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                     cudaStream_t s) {
    const dim3 grid((g.W + 31) / 32, max_chain_blocks<kChainR>(g, lt), nimg * lt.n);
    kz_launch(k_hess_det_chain<kChainR>, dim3(grid), dim3(dim3(32, 8)), 0, s, Lxy, Ldet, img_stride, g, lt);
}

bool launch_hess_fused(const float* Lt, float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg,
                       const LevelTable& lt, int keep_edges, cudaStream_t s) {
    int gx = 1, gy = 1;
    for (int l = 0; l < lt.n; ++l) {
        const int st = lt.step[l];
        if (st > 32) return false;  // CW + 2s > 256: the two-pass form handles it
        gx = max(gx, (g.W + fused_cw_host(st) - 1) / fused_cw_host(st));
        gy = max(gy, st * ((g.H + kFusedR * st - 1) / (kFusedR * st)));
    }
    kz_launch(k_hess_fused<kFusedR>, dim3(dim3(gx, gy, nimg * lt.n)), dim3(256), 0, s, Lt, Lxy, Ldet, img_stride, g, lt, keep_edges);
    return true;
}

void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s) {
    kz_launch(k_component_copy, dim3(dim3((g.W + 255) / 256, g.H)), dim3(256), 0, s, plane, comp, tight, to_tight, g);
}

}  // namespace kz
