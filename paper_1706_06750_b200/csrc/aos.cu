// aos.cu — semi-implicit AOS step of Eq. 4 (readings A1, A2) on sm_100a.
//
// L_i = ½[(I − 2τA_x(c))⁻¹ + (I − 2τA_y(c))⁻¹] L_{i−1}: H row systems of length W (k_aos_rows_cta → V, first) and
// W column systems of length H (k_cols_* → L_i = ½(U + V), second).  Every line is tridiagonal with
//   a_j = −τ(c_{j−1} + c_j),  cc_j = −τ(c_j + c_{j+1}),  b_j = 1 − a_j − cc_j   (Neumann ends: a_0 = cc_{n−1} = 0).
//
// Both passes use the partition ("Thomas–PCR hybrid") scheme of DESIGN.md §6: a line is cut into T chunks of M
// samples (the last takes the remainder, 2..M+1), one thread per chunk.  Each thread eliminates its chunk in
// registers (downward sweep keeping x_first, upward sweep keeping x_last), leaving x_i = δ'_i − α'_i x_first −
// γ'_i x_last and two reduced equations; substituting the neighbour's last equation gives a tridiagonal system in
// the T chunk-first unknowns; after it is solved every thread evaluates its samples.  One 1-ulp reciprocal per
// sample.
//   rows:    one CTA (4 or 8 warps) per row.  The TMA engine streams the row's L and c into shared memory (1-D bulk
//            copies, mbarrier), M is odd so the strided chunk reads are conflict free; the reduced system is solved
//            by a warp-level SPIKE (shuffle PCR on three right-hand sides + a 2·NW-unknown boundary solve), and V
//            leaves through shared memory with 16-byte stores.
//   columns: three register-light passes (k_cols_reduce / k_cols_solve / k_cols_final, see below): every warp
//            covers 32 adjacent columns, so every access is a full 128-byte row segment; no shared memory and no
//            barriers; L_i = ½(U + V) is written by the last pass.
#include "kaze_internal.cuh"
#include "ptx.cuh"

namespace kz {

namespace {

template <int MC>
struct Chunk {
    float al[MC], ga[MC], de[MC];  // α', γ', δ' of rows 1..m-2
    float A, C, D;                 // first equation (normalised)
    float lA, lG, lD;              // last equation  α x_first + x_last + γ x_next_first = δ
};

// dv[i] = L at sample j0+i, cv[i] = c at j0+i (i < m), cprev = c at j0-1, cnext = c at j0+m.
template <int MC>
__device__ __forceinline__ void eliminate(Chunk<MC>& ch, const float (&dv)[MC], const float (&cv)[MC], float cprev,
                                          float cnext, int m, bool first_chunk, bool last_chunk, float tau) {
    auto coef = [&](int i, float& a, float& b, float& cc) {
        const float cl = (i == 0) ? cprev : cv[i > 0 ? i - 1 : 0];
        const float cm = cv[i];
        const float cr = (i == m - 1) ? cnext : cv[i + 1 < MC ? i + 1 : MC - 1];
        a = (i == 0 && first_chunk) ? 0.f : -tau * (cl + cm);
        cc = (i == m - 1 && last_chunk) ? 0.f : -tau * (cm + cr);
        b = 1.f - a - cc;
    };
    // downward sweep (rows 1..m-1), virtual row 0: α = -1, γ = 0, δ = 0
    float pa = -1.f, pg = 0.f, pd = 0.f;
#pragma unroll
    for (int i = 1; i < MC; ++i) {
        if (i < m) {
            float a, b, cc;
            coef(i, a, b, cc);
            const float r = frcp(b - a * pg);
            const float na = -a * pa * r;
            const float ng = cc * r;
            const float nd = (dv[i] - a * pd) * r;
            ch.al[i] = na;
            ch.ga[i] = ng;
            ch.de[i] = nd;
            pa = na;
            pg = ng;
            pd = nd;
        }
    }
    ch.lA = pa;
    ch.lG = pg;
    ch.lD = pd;
    // upward sweep (rows m-2..1), virtual row m-1: α' = 0, γ' = -1, δ' = 0
    float na = 0.f, ng = -1.f, nd = 0.f;
#pragma unroll
    for (int i = MC - 2; i >= 1; --i) {
        if (i <= m - 2) {
            const float g = ch.ga[i];
            const float a2 = ch.al[i] - g * na;
            const float g2 = -g * ng;
            const float d2 = ch.de[i] - g * nd;
            ch.al[i] = a2;
            ch.ga[i] = g2;
            ch.de[i] = d2;
            na = a2;
            ng = g2;
            nd = d2;
        }
    }
    // row 0: a0 x_{-1} + b0 x0 + cc0 x1 = d0 with x1 = nd - na x0 - ng x_last
    float a0, b0, c0;
    coef(0, a0, b0, c0);
    const float rB = frcp(b0 - c0 * na);
    ch.A = a0 * rB;
    ch.C = -c0 * ng * rB;
    ch.D = (dv[0] - c0 * nd) * rB;
}

// Fast path for a full chunk of exactly M samples (every chunk but possibly the last): no per-sample predicates.
// tq[i] = τ(c_{i-1} + c_i) for i = 0..M (tq[0] uses c at j0-1, tq[M] c at j0+M; zeroed at the line ends), so
// a_i = -tq[i], cc_i = -tq[i+1], b_i = 1 + tq[i] + tq[i+1].
template <int M>
__device__ __forceinline__ void eliminate_full(Chunk<M + 1>& ch, const float (&dv)[M + 1], const float (&cv)[M + 1],
                                               float cprev, float cnext, bool first_chunk, bool last_chunk, float tau) {
    float tq[M + 1], bb[M];
    tq[0] = first_chunk ? 0.f : tau * (cprev + cv[0]);
#pragma unroll
    for (int i = 1; i < M; ++i) tq[i] = tau * (cv[i - 1] + cv[i]);
    tq[M] = last_chunk ? 0.f : tau * (cv[M - 1] + cnext);
#pragma unroll
    for (int i = 0; i < M; ++i) bb[i] = 1.f + tq[i] + tq[i + 1];
    float pa = -1.f, pg = 0.f, pd = 0.f;
#pragma unroll
    for (int i = 1; i < M; ++i) {
        const float r = frcp(fmaf(tq[i], pg, bb[i]));  // b_i - a_i γ_{i-1}
        const float na = tq[i] * pa * r;
        const float ng = -tq[i + 1] * r;
        const float nd = fmaf(tq[i], pd, dv[i]) * r;
        ch.al[i] = na;
        ch.ga[i] = ng;
        ch.de[i] = nd;
        pa = na;
        pg = ng;
        pd = nd;
    }
    ch.lA = pa;
    ch.lG = pg;
    ch.lD = pd;
    float na = 0.f, ng = -1.f, nd = 0.f;
#pragma unroll
    for (int i = M - 2; i >= 1; --i) {
        const float gi = ch.ga[i];
        const float a2 = ch.al[i] - gi * na;
        const float g2 = -gi * ng;
        const float d2 = ch.de[i] - gi * nd;
        ch.al[i] = a2;
        ch.ga[i] = g2;
        ch.de[i] = d2;
        na = a2;
        ng = g2;
        nd = d2;
    }
    // row 0: a0 = -tq[0], cc0 = -tq[1], b0 = bb[0]
    const float rB = frcp(fmaf(tq[1], na, bb[0]));
    ch.A = -tq[0] * rB;
    ch.C = tq[1] * ng * rB;
    ch.D = fmaf(tq[1], nd, dv[0]) * rB;
}

// Chunking of a line of n samples into chunks of M: T chunks, chunk p = [p*M, p*M + size), the last one takes the
// remainder; a remainder of 1 is merged into the previous chunk (so 2 <= size <= M+1).
__host__ __device__ inline int n_chunks(int n, int M) {
    int T = (n + M - 1) / M;
    if (T > 1 && n - (T - 1) * M == 1) --T;
    return T;
}

// -------------------------------------------------------------------------------------------------------------
// Column systems in three register-light passes (no shared memory, no barriers, every warp = 32 adjacent columns,
// so every access is a full 128-byte row segment):
//   cols_reduce : per (column, chunk of M rows): a downward sweep keeping x_first gives the chunk's LAST equation
//                 α x_first + x_last + γ x_next = δ, a mirrored upward sweep keeping x_last gives its FIRST equation
//                 x_first + α~ x_prev + γ~ x_last = δ~ (O(1) state each, the chunk's L and c held in registers).
//   cols_solve  : per column, the 2T reduced unknowns (x_first, x_last of every chunk) form a tridiagonal system,
//                 solved by Thomas (diagonally dominant: Schur complement of an M-matrix).
//   cols_final  : per chunk, the interior with known end values is a plain Thomas solve; L_i = ½(U + V) is written.
// DRAM traffic stays at the algorithmic 16 B/px when the level's L and c stay in L2 between the first and last
// pass (they are re-read there).
template <int M>
__global__ void __launch_bounds__(256) k_cols_reduce(const float* __restrict__ L, const float* __restrict__ c,
                                                     float* __restrict__ red, Strides st, Geom g, float tau, int T,
                                                     size_t red_img_stride) {
    constexpr int MC = M + 1;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const int p = blockIdx.y * 8 + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= g.W || p >= T) return;
    const int n = g.H;
    const int j0 = p * M, j1 = (p == T - 1) ? n : j0 + M, m = j1 - j0;
    const float* Lc = L + z * st.L + (size_t)j0 * g.P + x;
    const float* cc = c + z * st.c + (size_t)j0 * g.P + x;
    float dv[MC], tq[MC + 1];  // tq[i] = τ(c_{i-1} + c_i) for i = 0..m (0 at the line ends)
    float cv[MC];
    const uint64_t keep = l2_policy_evict_last();  // L and c are read again by k_cols_final: keep them in L2
#pragma unroll
    for (int i = 0; i < MC; ++i) {
        dv[i] = i < m ? ld_policy(Lc + (size_t)i * g.P, keep) : 0.f;
        cv[i] = i < m ? ld_policy(cc + (size_t)i * g.P, keep) : 0.f;
    }
    const float cprev = j0 > 0 ? __ldg(cc - g.P) : 0.f;
    const float cnext = j1 < n ? __ldg(cc + (size_t)m * g.P) : 0.f;
    tq[0] = j0 > 0 ? tau * (cprev + cv[0]) : 0.f;
#pragma unroll
    for (int i = 1; i <= MC; ++i) {
        float v;
        if (i < m) v = tau * (cv[i - 1] + cv[i]);
        else if (i == m) v = j1 < n ? tau * (cv[i - 1 < MC ? i - 1 : 0] + cnext) : 0.f;
        else v = 0.f;
        tq[i] = v;
    }
    // row i: a_i = -tq[i], cc_i = -tq[i+1], b_i = 1 + tq[i] + tq[i+1]
    float pa = -1.f, pg = 0.f, pd = 0.f;  // downward, virtual row 0
#pragma unroll
    for (int i = 1; i < MC; ++i) {
        if (i < m) {
            const float r = frcp(1.f + tq[i] + tq[i + 1] + tq[i] * pg);
            pa = tq[i] * pa * r;
            pg = -tq[i + 1] * r;
            pd = fmaf(tq[i], pd, dv[i]) * r;
        }
    }
    float qa = 0.f, qg = -1.f, qd = 0.f;  // upward, virtual row m-1: x_i + qa x_{i-1} + qg x_last = qd
#pragma unroll
    for (int i = MC - 1; i >= 0; --i) {
        if (i <= m - 2) {
            const float r = frcp(1.f + tq[i] + tq[i + 1] + tq[i + 1] * qa);  // b_i - cc_i α~_{i+1}
            qa = -tq[i] * r;
            qg = tq[i + 1] * qg * r;
            qd = fmaf(tq[i + 1], qd, dv[i]) * r;
        }
    }
    // [z][p][6][W]: first (α~, γ~, δ~), last (α, γ, δ)
    float* o = red + z * red_img_stride + (size_t)p * 6 * g.W + x;
    o[0] = qa;
    o[(size_t)g.W] = qg;
    o[(size_t)2 * g.W] = qd;
    o[(size_t)3 * g.W] = pa;
    o[(size_t)4 * g.W] = pg;
    o[(size_t)5 * g.W] = pd;
}

// One thread per column: Thomas on u = (f_0, l_0, f_1, l_1, ...),
//   f_p:  α~_p l_{p-1} + f_p + γ~_p l_p = δ~_p,      l_p:  α_p f_p + l_p + γ_p f_{p+1} = δ_p.
// The forward sweep's (c', d') are kept in the output slots; the backward sweep overwrites them with u.
__global__ void __launch_bounds__(128) k_cols_solve(float* __restrict__ red, float* __restrict__ sol, Geom g, int T,
                                                    size_t red_img_stride, size_t sol_img_stride) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, z = blockIdx.y;
    if (x >= g.W) return;
    const float* e = red + z * red_img_stride + x;
    float* u = sol + z * sol_img_stride + x;  // [z][2T][2][W]: (c', d') then u
    const size_t W = g.W;
    // the coefficients of 4 chunks (8 equations) are fetched one batch ahead of the recurrence
    constexpr int KB = 4;
    float cur[KB * 6], nxt[KB * 6];
#pragma unroll
    for (int i = 0; i < KB * 6; ++i) cur[i] = (i / 6) < T ? __ldg(e + (size_t)i * W) : 0.f;
    float cp = 0.f, dp = 0.f;
    for (int p0 = 0; p0 < T; p0 += KB) {
#pragma unroll
        for (int i = 0; i < KB * 6; ++i) nxt[i] = (p0 + KB + i / 6) < T ? __ldg(e + (size_t)(p0 * 6 + KB * 6 + i) * W) : 0.f;
#pragma unroll
        for (int q = 0; q < KB; ++q) {
            if (p0 + q < T) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // f then l equation of chunk p0+q
                    const float sub = cur[q * 6 + 3 * h], sup = cur[q * 6 + 3 * h + 1], rhs = cur[q * 6 + 3 * h + 2];
                    const float r = frcp(1.f - sub * cp);
                    cp = sup * r;
                    dp = (rhs - sub * dp) * r;
                    const size_t k = (size_t)(2 * (p0 + q) + h);
                    u[k * 2 * W] = cp;
                    u[k * 2 * W + W] = dp;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < KB * 6; ++i) cur[i] = nxt[i];
    }
    // backward: u_k = d'_k - c'_k u_{k+1}; the (c', d') pairs are re-read a batch ahead as well
    float xn = 0.f;
    for (int k0 = 2 * T - 1; k0 >= 0; k0 -= 8) {
        float cc8[8], dd8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 - i;
            cc8[i] = k >= 0 ? u[(size_t)k * 2 * W] : 0.f;
            dd8[i] = k >= 0 ? u[(size_t)k * 2 * W + W] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 - i;
            if (k >= 0) {
                xn = dd8[i] - cc8[i] * xn;
                u[(size_t)k * 2 * W + W] = xn;
            }
        }
    }
}

template <int M>
__global__ void __launch_bounds__(256) k_cols_final(const float* __restrict__ L, const float* __restrict__ c,
                                                    const float* __restrict__ V, const float* __restrict__ sol,
                                                    float* __restrict__ Lout, Strides st, Geom g, float tau, int T,
                                                    size_t sol_img_stride) {
    constexpr int MC = M + 1;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const int p = blockIdx.y * 8 + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= g.W || p >= T) return;
    const int n = g.H;
    const int j0 = p * M, j1 = (p == T - 1) ? n : j0 + M, m = j1 - j0;
    const size_t W = g.W;
    const float* u = sol + z * sol_img_stride + x;
    const float xf = u[(size_t)(2 * p) * 2 * W + W], xl = u[(size_t)(2 * p + 1) * 2 * W + W];
    const float* Lc = L + z * st.L + (size_t)j0 * g.P + x;
    const float* cc = c + z * st.c + (size_t)j0 * g.P + x;
    const float* Vc = V + z * st.U + (size_t)j0 * g.P + x;
    float dv[MC], cv[MC], vv[MC];
    const uint64_t done = l2_policy_evict_first();  // last use of this level's L, c and V
#pragma unroll
    for (int i = 0; i < MC; ++i) {
        dv[i] = i < m ? ld_policy(Lc + (size_t)i * g.P, done) : 0.f;
        cv[i] = i < m ? ld_policy(cc + (size_t)i * g.P, done) : 0.f;
        vv[i] = i < m ? ld_policy(Vc + (size_t)i * g.P, done) : 0.f;
    }
    // interior rows 1..m-2 with x_0 = xf and x_{m-1} = xl known; τ(c_{i-1}+c_i) for i = 1..m-1 (interior only)
    float cpv[MC], dpv[MC];
    float cp = 0.f, dp = 0.f;
#pragma unroll
    for (int i = 1; i < MC; ++i) {
        if (i <= m - 2) {
            const float ta = tau * (cv[i - 1] + cv[i]), tb = tau * (cv[i] + cv[i + 1 < MC ? i + 1 : 0]);
            float rhs = dv[i];
            if (i == 1) rhs += ta * xf;          // -a_1 x_0
            if (i == m - 2) rhs += tb * xl;      // -cc_{m-2} x_{m-1}
            const float sub = (i == 1) ? 0.f : -ta;
            const float sup = (i == m - 2) ? 0.f : -tb;
            const float r = frcp(1.f + ta + tb - sub * cp);
            cp = sup * r;
            dp = (rhs - sub * dp) * r;
            cpv[i] = cp;
            dpv[i] = dp;
        }
    }
    float* Oc = Lout + z * st.out + (size_t)j0 * g.P + x;
    float xn = xl;
#pragma unroll
    for (int i = MC - 1; i >= 0; --i) {
        if (i == m - 1) Oc[(size_t)i * g.P] = 0.5f * (xl + vv[i]);
        else if (i >= 1 && i <= m - 2) {
            xn = dpv[i] - cpv[i] * xn;
            Oc[(size_t)i * g.P] = 0.5f * (xn + vv[i]);
        }
    }
    Oc[0] = 0.5f * (xf + vv[0]);
}

// -------------------------------------------------------------------------------------------------------------
// Row systems, one CTA of NW warps per row (the row pass runs first and writes V).  The TMA engine streams the
// row's L and c into shared memory; thread p owns the chunk [p·M, p·M + m) (M odd: conflict-free strided reads)
// and eliminates it in registers; the reduced system (one unknown per thread) is solved by a warp-level SPIKE:
// shuffle PCR inside each warp on three right-hand sides, a serial 2·NW-unknown boundary solve by one thread,
// then x = y − v·x_{prev warp} − z·x_{next warp}.  x goes back to shared memory and V leaves with 16-byte stores.
template <int M, int NW>
__global__ void __launch_bounds__(32 * NW) k_aos_rows_cta(const float* __restrict__ L, const float* __restrict__ c,
                                                          float* __restrict__ V, Strides st, Geom g, float tau, int T) {
    constexpr int MC = M + 1, TP = 32 * NW;
    extern __shared__ __align__(16) float rs[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ float lastA[TP], lastG[TP], lastD[TP], bnd[NW * 6], sol[NW * 2], fx[TP];
    const int n = g.W;
    const int Wp = (n + 3) & ~3;
    float* sL = rs;
    float* sC = rs + Wp;
    const int p = threadIdx.x, lane = p & 31, w = p >> 5;
    const int img = blockIdx.x / g.H, y = blockIdx.x - img * g.H;
    const size_t ry = (size_t)y * g.P;
    if (p == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 8u * (uint32_t)Wp);
        bulk_g2s(sL, L + img * st.L + ry, 4u * (uint32_t)Wp, &bar);
        bulk_g2s(sC, c + img * st.c + ry, 4u * (uint32_t)Wp, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    const bool active = p < T;
    const int j0 = p * M;
    const int j1 = (p == T - 1) ? n : j0 + M;
    const int m = active ? j1 - j0 : 0;
    Chunk<MC> ch;
    if (active) {
        float dv[MC], cv[MC];
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            dv[i] = i < m ? sL[j0 + i] : 0.f;
            cv[i] = i < m ? sC[j0 + i] : 0.f;
        }
        const float cprev = p > 0 ? sC[j0 - 1] : 0.f;
        const float cnext = j1 < n ? sC[j1] : 0.f;
        if (m == M) eliminate_full<M>(ch, dv, cv, cprev, cnext, p == 0, p == T - 1, tau);
        else eliminate<MC>(ch, dv, cv, cprev, cnext, m, p == 0, p == T - 1, tau);
    } else {
        ch.A = ch.C = ch.D = 0.f;
        ch.lA = ch.lG = ch.lD = 0.f;
    }
    lastA[p] = ch.lA;
    lastG[p] = ch.lG;
    lastD[p] = ch.lD;
    __syncthreads();
    float a = 0.f, b = 1.f, cc = 0.f, r0 = 0.f;
    if (active) {
        const float pA = p > 0 ? lastA[p - 1] : 0.f, pG = p > 0 ? lastG[p - 1] : 0.f, pD = p > 0 ? lastD[p - 1] : 0.f;
        a = -ch.A * pA;
        b = 1.f - ch.A * pG - ch.C * ch.lA;
        cc = -ch.C * ch.lG;
        r0 = ch.D - ch.A * pD - ch.C * ch.lD;
    }
    // --- warp SPIKE: local block solve with couplings to the neighbouring warps moved to two extra RHS ---
    float r1 = 0.f, r2 = 0.f;
    if (lane == 0) {
        r1 = a;
        a = 0.f;
    }
    if (lane == 31) {
        r2 = cc;
        cc = 0.f;
    }
#pragma unroll
    for (int s2 = 1; s2 < 32; s2 <<= 1) {
        const bool hm = lane >= s2, hp = lane + s2 < 32;
        const float am = __shfl_up_sync(0xffffffffu, a, s2), bm = __shfl_up_sync(0xffffffffu, b, s2);
        const float cm = __shfl_up_sync(0xffffffffu, cc, s2), q0m = __shfl_up_sync(0xffffffffu, r0, s2);
        const float q1m = __shfl_up_sync(0xffffffffu, r1, s2), q2m = __shfl_up_sync(0xffffffffu, r2, s2);
        const float ap = __shfl_down_sync(0xffffffffu, a, s2), bp = __shfl_down_sync(0xffffffffu, b, s2);
        const float cp = __shfl_down_sync(0xffffffffu, cc, s2), q0p = __shfl_down_sync(0xffffffffu, r0, s2);
        const float q1p = __shfl_down_sync(0xffffffffu, r1, s2), q2p = __shfl_down_sync(0xffffffffu, r2, s2);
        const float k1 = hm ? a * frcp(bm) : 0.f;
        const float k2 = hp ? cc * frcp(bp) : 0.f;
        a = hm ? -am * k1 : 0.f;
        cc = hp ? -cp * k2 : 0.f;
        b = b - (hm ? cm * k1 : 0.f) - (hp ? ap * k2 : 0.f);
        r0 = r0 - (hm ? q0m * k1 : 0.f) - (hp ? q0p * k2 : 0.f);
        r1 = r1 - (hm ? q1m * k1 : 0.f) - (hp ? q1p * k2 : 0.f);
        r2 = r2 - (hm ? q2m * k1 : 0.f) - (hp ? q2p * k2 : 0.f);
    }
    const float rb = frcp(b);
    const float yv = r0 * rb, vv = r1 * rb, zv = r2 * rb;
    if (lane == 0 || lane == 31) {
        float* o = bnd + w * 6 + (lane == 0 ? 0 : 3);
        o[0] = yv;
        o[1] = vv;
        o[2] = zv;
    }
    __syncthreads();
    if (p == 0) {  // F_w = y0 - v0 G_{w-1} - z0 F_{w+1},  G_w = y31 - v31 G_{w-1} - z31 F_{w+1}
        float phi[NW], psi[NW], gam[NW], mu[NW];
        float gp = 0.f, mp = 0.f;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const float* o = bnd + k * 6;
            const float rden = frcp(1.f - o[1] * mp);
            phi[k] = (o[0] - o[1] * gp) * rden;
            psi[k] = o[2] * rden;
            gam[k] = o[3] - o[4] * gp + o[4] * mp * phi[k];
            mu[k] = o[4] * mp * psi[k] + o[5];
            gp = gam[k];
            mp = mu[k];
        }
        float Fn = 0.f;
#pragma unroll
        for (int k = NW - 1; k >= 0; --k) {
            sol[2 * k + 1] = gam[k] - mu[k] * Fn;
            Fn = phi[k] - psi[k] * Fn;
            sol[2 * k] = Fn;
        }
    }
    __syncthreads();
    const float xf = yv - vv * (w > 0 ? sol[2 * w - 1] : 0.f) - zv * (w + 1 < NW ? sol[2 * w + 2] : 0.f);
    fx[p] = xf;
    __syncthreads();
    if (active) {
        const float xnext = (p + 1 < T) ? fx[p + 1] : 0.f;
        const float xl = ch.lD - ch.lA * xf - ch.lG * xnext;
        sL[j0] = xf;
#pragma unroll
        for (int i = 1; i < MC; ++i)
            if (i < m - 1) sL[j0 + i] = ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl;
        sL[j1 - 1] = xl;
    }
    __syncthreads();
    float4* Vr = reinterpret_cast<float4*>(V + img * st.out + ry);
    for (int v = p; v < (Wp >> 2); v += TP) Vr[v] = reinterpret_cast<const float4*>(sL)[v];
}

template <int M, int NW>
void run_rows_cta(const float* L, const float* c, float* V, Strides st, Geom g, int nimg, float tau, cudaStream_t s) {
    int T = (g.W + M - 1) / M;
    if (T > 1 && g.W - (T - 1) * M == 1) --T;
    const size_t smem = sizeof(float) * 2 * ((g.W + 3) & ~3);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_aos_rows_cta<M, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    k_aos_rows_cta<M, NW><<<g.H * nimg, 32 * NW, smem, s>>>(L, c, V, st, g, tau, T);
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

}  // namespace

template <int M>
void run_cols3(const float* L, const float* c, const float* V, float* Lout, Strides st, Geom g, int nimg, float tau,
               float* red, float* sol, cudaStream_t s) {
    const int T = n_chunks(g.H, M);
    const size_t red_stride = (size_t)T * 6 * g.W, sol_stride = (size_t)T * 4 * g.W;
    dim3 blk(32, 8), grd((g.W + 31) / 32, (T + 7) / 8, nimg);
    k_cols_reduce<M><<<grd, blk, 0, s>>>(L, c, red, st, g, tau, T, red_stride);
    k_cols_solve<<<dim3((g.W + 127) / 128, nimg), 128, 0, s>>>(red, sol, g, T, red_stride, sol_stride);
    k_cols_final<M><<<grd, blk, 0, s>>>(L, c, V, sol, Lout, st, g, tau, T, sol_stride);
}

// Columns: three-pass register-light scheme (chunk M = 16 rows, 8 for short columns).  red / sol: scratch of at
// least 6·T·W and 4·T·W floats per image.
bool launch_aos_cols(const float* L, const float* c, const float* V, float* Lout, Strides st, Geom g, int nimg,
                     float tau, float* red, float* sol, cudaStream_t s) {
    if (g.H >= 256) run_cols3<16>(L, c, V, Lout, st, g, nimg, tau, red, sol, s);
    else run_cols3<8>(L, c, V, Lout, st, g, nimg, tau, red, sol, s);
    return true;
}

// Row systems, one CTA per row: the smallest odd chunk M >= 5 with T = ceil(W/M) <= 32·NW threads.
bool launch_aos_rows(const float* L, const float* c, float* V, Strides st, Geom g, int nimg, float tau,
                     cudaStream_t s) {
    const int W = g.W;
    if (W <= 128 * 5) run_rows_cta<5, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 128 * 7) run_rows_cta<7, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 128 * 9) run_rows_cta<9, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 128 * 11) run_rows_cta<11, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 128 * 13) run_rows_cta<13, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 128 * 15) run_rows_cta<15, 4>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 256 * 11) run_rows_cta<11, 8>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 256 * 17) run_rows_cta<17, 8>(L, c, V, st, g, nimg, tau, s);
    else if (W <= 256 * 33) run_rows_cta<33, 8>(L, c, V, st, g, nimg, tau, s);
    else return false;
    return true;
}

}  // namespace kz
