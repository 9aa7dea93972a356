// aos.cu — semi-implicit AOS step of Eq. 4 (readings A1, A2) on sm_100a.
//
// L_i = ½[(I − 2τA_y(c))⁻¹ + (I − 2τA_x(c))⁻¹] L_{i−1}: W column systems of length H (k_aos_cols → U) and
// H row systems of length W (k_aos_rows → L_i = ½(U + V)).  Every line is tridiagonal with
//   a_j = −τ(c_{j−1} + c_j),  cc_j = −τ(c_j + c_{j+1}),  b_j = 1 − a_j − cc_j   (Neumann ends: a_0 = cc_{n−1} = 0).
//
// Parallel scheme (partition / "Thomas–PCR hybrid"): a line of n samples is cut into T chunks of M
// samples (the last chunk takes the remainder, 2..M+1 samples), one thread per chunk.  Each thread
//   1. eliminates its chunk in registers (downward sweep keeping x_first, then upward sweep keeping x_last), so
//      every interior sample reads x_i = δ'_i − α'_i x_first − γ'_i x_last, and the chunk contributes two
//      reduced equations: F_p: A x_{last,p−1} + x_{first,p} + C x_{last,p} = D,
//                         L_p: α x_{first,p} + x_{last,p} + γ x_{first,p+1} = δ;
//   2. substitutes L_{p−1}, L_p into F_p → a tridiagonal system in the T unknowns x_{first,p}, solved by parallel
//      cyclic reduction in shared memory (⌈log2 T⌉ steps);
//   3. evaluates its samples from the two chunk-end values.
// One (approximate, 1-ulp) reciprocal per sample.  Column lines are read straight from global memory (a warp covers
// CW adjacent columns × 32/CW chunks: every request is whole 32-byte sectors).  Row lines are staged through shared
// memory with coalesced 16-byte loads; the chunk length M is odd so the per-thread sweeps (stride M) are
// bank-conflict free.
#include "kaze_internal.cuh"
#include "ptx.cuh"

namespace kz {

namespace {

// Parallel cyclic reduction of a tridiagonal system with one equation per thread (p = 0..TP-1 within its
// system, idx = p*stride + off in the shared arrays).  Threads p >= T carry identity rows.  Returns x_p.
__device__ __forceinline__ float pcr_solve(float af, float bf, float cf, float df, int p, int TP, int stride, int idx,
                                           float* sa, float* sb, float* sc, float* sd) {
    for (int st = 1; st < TP; st <<= 1) {
        sa[idx] = af;
        sb[idx] = bf;
        sc[idx] = cf;
        sd[idx] = df;
        __syncthreads();
        const bool hm = p >= st, hp = p + st < TP;
        const int jm = hm ? idx - st * stride : idx, jp = hp ? idx + st * stride : idx;
        const float am = sa[jm], bm = sb[jm], cm = sc[jm], dm = sd[jm];
        const float ap = sa[jp], bp = sb[jp], cp = sc[jp], dp = sd[jp];
        const float k1 = hm ? af * frcp(bm) : 0.f;
        const float k2 = hp ? cf * frcp(bp) : 0.f;
        __syncthreads();
        af = -am * k1;
        cf = -cp * k2;
        bf = bf - cm * k1 - ap * k2;
        df = df - dm * k1 - dp * k2;
    }
    return df * frcp(bf);
}

// Warp-level SPIKE solve of NS independent tridiagonal systems of TP equations (TP % 32 == 0, TP/32 <= 8) that
// the CTA holds one equation per thread.  Threads are re-mapped so each warp owns 32 consecutive equations of one
// system: the warp solves its 32x32 block for the right-hand side and the two coupling columns by PCR over
// shuffles (5 steps, no barriers); one thread per system then solves the 2·(TP/32) warp-boundary unknowns by a
// serial block recursion, and every equation reads x = y − v·x_{prev warp last} − z·x_{next warp first}.
// Four block barriers in total (against 2·⌈log2 TP⌉ for a shared-memory PCR).  Returns the calling thread's x.
// Scratch: e* [NS][TP+1], bnd [NS][8][6], sol [NS][8][2].
__device__ __forceinline__ float spike_solve(float af, float bf, float cf, float df, int s, int p, int NS, int TP,
                                             float* ea, float* eb, float* ec, float* ed, float* bnd, float* sol) {
    const int SP = TP + 1;
    ea[s * SP + p] = af;
    eb[s * SP + p] = bf;
    ec[s * SP + p] = cf;
    ed[s * SP + p] = df;
    __syncthreads();
    const int t = threadIdx.x;
    const int s2 = t / TP, p2 = t - s2 * TP;
    const int lane = t & 31, w = p2 >> 5, nw = TP >> 5;
    const bool live = s2 < NS;
    float a = 0.f, b = 1.f, c = 0.f, r0 = 0.f, r1 = 0.f, r2 = 0.f;
    if (live) {
        const int i2 = s2 * SP + p2;
        a = ea[i2];
        b = eb[i2];
        c = ec[i2];
        r0 = ed[i2];
        if (lane == 0) {
            r1 = a;  // coupling to the previous warp's last unknown → right-hand side v
            a = 0.f;
        }
        if (lane == 31) {
            r2 = c;  // coupling to the next warp's first unknown → right-hand side z
            c = 0.f;
        }
    }
#pragma unroll
    for (int st = 1; st < 32; st <<= 1) {
        const bool hm = lane >= st, hp = lane + st < 32;
        float am = __shfl_up_sync(0xffffffffu, a, st), bm = __shfl_up_sync(0xffffffffu, b, st);
        float cm = __shfl_up_sync(0xffffffffu, c, st), q0m = __shfl_up_sync(0xffffffffu, r0, st);
        float q1m = __shfl_up_sync(0xffffffffu, r1, st), q2m = __shfl_up_sync(0xffffffffu, r2, st);
        float ap = __shfl_down_sync(0xffffffffu, a, st), bp = __shfl_down_sync(0xffffffffu, b, st);
        float cp = __shfl_down_sync(0xffffffffu, c, st), q0p = __shfl_down_sync(0xffffffffu, r0, st);
        float q1p = __shfl_down_sync(0xffffffffu, r1, st), q2p = __shfl_down_sync(0xffffffffu, r2, st);
        const float k1 = hm ? a * frcp(bm) : 0.f;
        const float k2 = hp ? c * frcp(bp) : 0.f;
        a = hm ? -am * k1 : 0.f;
        c = hp ? -cp * k2 : 0.f;
        b = b - (hm ? cm * k1 : 0.f) - (hp ? ap * k2 : 0.f);
        r0 = r0 - (hm ? q0m * k1 : 0.f) - (hp ? q0p * k2 : 0.f);
        r1 = r1 - (hm ? q1m * k1 : 0.f) - (hp ? q1p * k2 : 0.f);
        r2 = r2 - (hm ? q2m * k1 : 0.f) - (hp ? q2p * k2 : 0.f);
    }
    const float rb = frcp(b);
    const float y = r0 * rb, v = r1 * rb, z = r2 * rb;
    if (live && (lane == 0 || lane == 31)) {
        float* o = bnd + ((s2 * 8 + w) * 6 + (lane == 0 ? 0 : 3));
        o[0] = y;
        o[1] = v;
        o[2] = z;
    }
    __syncthreads();
    if (live && p2 == 0) {  // F_w = y0 - v0 G_{w-1} - z0 F_{w+1},  G_w = y31 - v31 G_{w-1} - z31 F_{w+1}
        float o[8][6];          // all boundary data loaded up front (one shared-memory latency, not eight)
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int e = 0; e < 6; ++e) o[k][e] = k < nw ? bnd[(s2 * 8 + k) * 6 + e] : 0.f;
        float phi[8], psi[8], gam[8], mu[8];
        float gp = 0.f, mp = 0.f;  // G_{w-1} = gp - mp F_w
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float rden = frcp(1.f - o[k][1] * mp);
            phi[k] = (o[k][0] - o[k][1] * gp) * rden;
            psi[k] = o[k][2] * rden;
            gam[k] = o[k][3] - o[k][4] * gp + o[k][4] * mp * phi[k];
            mu[k] = o[k][4] * mp * psi[k] + o[k][5];
            gp = gam[k];
            mp = mu[k];
        }
        float Fn = 0.f;
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            if (k < nw) {
                sol[(s2 * 8 + k) * 2 + 1] = gam[k] - mu[k] * Fn;
                Fn = phi[k] - psi[k] * Fn;
                sol[(s2 * 8 + k) * 2 + 0] = Fn;
            }
        }
    }
    __syncthreads();
    if (live) {
        const float Gprev = w > 0 ? sol[(s2 * 8 + w - 1) * 2 + 1] : 0.f;
        const float Fnext = w + 1 < nw ? sol[(s2 * 8 + w + 1) * 2 + 0] : 0.f;
        ed[s2 * SP + p2] = y - v * Gprev - z * Fnext;
    }
    __syncthreads();
    return ed[s * SP + p];
}

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
// Column systems.  Thread (cx, p): column x0 + cx, chunk p of T.  blockDim.x = CW * TP; shared index p*CW + cx.
template <int CW, int M, int NT>
__global__ void __launch_bounds__(NT) k_aos_cols(const float* __restrict__ L, const float* __restrict__ c,
                                                 const float* __restrict__ U, float* __restrict__ Lout, Strides st,
                                                 Geom g, float tau, int T, int TP) {
    constexpr int MC = M + 1;
    extern __shared__ float sm[];
    const int NTOT = CW * TP;
    float* sa = sm;
    float* sb = sa + NTOT;
    float* sc = sb + NTOT;
    float* sd = sc + NTOT;
    float* sla = sd + NTOT;  // last-equation exchange
    float* slg = sla + NTOT;
    float* sld = slg + NTOT;
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int x = blockIdx.x * CW + cx;
    const bool active = (p < T) && (x < g.W);
    const int n = g.H;
    const int j0 = p * M;
    const int j1 = (p == T - 1) ? n : j0 + M;
    const int m = active ? j1 - j0 : 0;

    Chunk<MC> ch;
    if (active) {
        float dv[MC], cv[MC];
        const float* Lc = L + blockIdx.z * st.L + (size_t)j0 * g.P + x;
        const float* cc = c + blockIdx.z * st.c + (size_t)j0 * g.P + x;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            if (i < m) {
                dv[i] = __ldg(Lc + (size_t)i * g.P);
                cv[i] = __ldg(cc + (size_t)i * g.P);
            } else {
                dv[i] = 0.f;
                cv[i] = 0.f;
            }
        }
        const float cprev = j0 > 0 ? __ldg(cc - g.P) : 0.f;
        const float cnext = j1 < n ? __ldg(cc + (size_t)m * g.P) : 0.f;
        if (m == M) eliminate_full<M>(ch, dv, cv, cprev, cnext, j0 == 0, j1 == n, tau);
        else eliminate<MC>(ch, dv, cv, cprev, cnext, m, j0 == 0, j1 == n, tau);
    } else {
        ch.A = ch.C = ch.D = 0.f;
        ch.lA = ch.lG = ch.lD = 0.f;
    }
    const int idx = p * CW + cx;
    sla[idx] = ch.lA;
    slg[idx] = ch.lG;
    sld[idx] = ch.lD;
    __syncthreads();
    float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
    if (active) {
        float pA = 0.f, pG = 0.f, pD = 0.f;
        if (p > 0) {
            pA = sla[idx - CW];
            pG = slg[idx - CW];
            pD = sld[idx - CW];
        }
        af = -ch.A * pA;
        bf = 1.f - ch.A * pG - ch.C * ch.lA;
        cf = -ch.C * ch.lG;
        df = ch.D - ch.A * pD - ch.C * ch.lD;
    }
    const float xf = pcr_solve(af, bf, cf, df, p, TP, CW, idx, sa, sb, sc, sd);
    sa[idx] = xf;
    __syncthreads();
    if (!active) return;
    const float xnext = (p + 1 < T) ? sa[idx + CW] : 0.f;
    const float xl = ch.lD - ch.lA * xf - ch.lG * xnext;
    // L_i = ½(U + V): the row pass already wrote V (passed in as U's buffer); the average is formed here.
    const float* Vc = U + blockIdx.z * st.U + (size_t)j0 * g.P + x;
    float* Oc = Lout + blockIdx.z * st.out + (size_t)j0 * g.P + x;
    Oc[0] = 0.5f * (xf + __ldg(Vc));
#pragma unroll
    for (int i = 1; i < MC; ++i) {
        if (i < m - 1) Oc[(size_t)i * g.P] = 0.5f * (ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl + __ldg(Vc + (size_t)i * g.P));
    }
    Oc[(size_t)(m - 1) * g.P] = 0.5f * (xl + __ldg(Vc + (size_t)(m - 1) * g.P));
}

// -------------------------------------------------------------------------------------------------------------
// Row systems: a persistent CTA walks rows q = blockIdx.x, +gridDim.x, ... of all images.  Each row's L, c and U
// are fetched by the TMA engine (1-D bulk copies, one mbarrier per stage) into a double-buffered shared stage, so
// the next row streams in while the current one is solved.  The row is solved from shared memory (contiguous
// layout; M odd → stride-M sweeps are conflict free), x overwrites L in place, and L_i = ½(U + x) is written with
// coalesced 16-byte stores.
template <int M>
__global__ void __launch_bounds__(256) k_aos_rows(const float* __restrict__ L, const float* __restrict__ c,
                                                  const float* __restrict__ U, float* __restrict__ Lout, Strides st,
                                                  Geom g, float tau, int T, int TP, int total_rows) {
    static_assert(M % 2 == 1, "row chunks must have odd length");
    constexpr int MC = M + 1;
    extern __shared__ __align__(128) float smf[];
    const int n = g.W;
    const int Wp = (n + 3) & ~3;              // row floats fetched (16-byte multiple; stays inside the pitch)
    float* stage = smf;                        // [2][3][Wp]: L, c, U
    float* sa = stage + 6 * Wp;                // SPIKE arrays [TP+1] each, boundary data, last-equation exchange
    float* sb = sa + (TP + 1);
    float* sc = sb + (TP + 1);
    float* sd = sc + (TP + 1);
    float* bnd = sd + (TP + 1);
    float* sol = bnd + 48;
    float* sla = sol + 16;
    float* slg = sla + TP;
    float* sld = slg + TP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(sld + TP + 1) & ~uintptr_t(7));
    const int tid = threadIdx.x;
    const uint32_t bytes = (uint32_t)Wp * 4u;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int q, int sidx) {
        const int img = q / g.H, y = q - img * g.H;
        const size_t ry = (size_t)y * g.P;
        float* dst = stage + sidx * 3 * Wp;
        mbar_arrive_expect_tx(&bar[sidx], 3u * bytes);
        bulk_g2s(dst, L + img * st.L + ry, bytes, &bar[sidx]);
        bulk_g2s(dst + Wp, c + img * st.c + ry, bytes, &bar[sidx]);
        bulk_g2s(dst + 2 * Wp, U + img * st.U + ry, bytes, &bar[sidx]);
    };
    int q = blockIdx.x;
    if (tid == 0 && q < total_rows) issue(q, 0);
    const int p = tid;
    const bool active = p < T;
    const int j0 = p * M;
    const int j1 = (p == T - 1) ? n : j0 + M;
    const int m = active ? j1 - j0 : 0;
    for (int it = 0; q < total_rows; ++it, q += gridDim.x) {
        const int sidx = it & 1;
        if (tid == 0 && q + (int)gridDim.x < total_rows) issue(q + gridDim.x, sidx ^ 1);
        mbar_wait(&bar[sidx], (uint32_t)(it >> 1) & 1u);
        float* sL = stage + sidx * 3 * Wp;
        const float* sC = sL + Wp;
        const float* sU = sL + 2 * Wp;
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
        sla[p] = ch.lA;
        slg[p] = ch.lG;
        sld[p] = ch.lD;
        __syncthreads();
        float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
        if (active) {
            float pA = 0.f, pG = 0.f, pD = 0.f;
            if (p > 0) {
                pA = sla[p - 1];
                pG = slg[p - 1];
                pD = sld[p - 1];
            }
            af = -ch.A * pA;
            bf = 1.f - ch.A * pG - ch.C * ch.lA;
            cf = -ch.C * ch.lG;
            df = ch.D - ch.A * pD - ch.C * ch.lD;
        }
        const float xf = spike_solve(af, bf, cf, df, 0, p, 1, TP, sa, sb, sc, sd, bnd, sol);
        if (active) {
            const float xnext = (p + 1 < T) ? sd[p + 1] : 0.f;
            const float xl = ch.lD - ch.lA * xf - ch.lG * xnext;
            sL[j0] = xf;
#pragma unroll
            for (int i = 1; i < MC; ++i)
                if (i < m - 1) sL[j0 + i] = ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl;
            sL[j1 - 1] = xl;
        }
        __syncthreads();
        {
            const int img = q / g.H, y = q - img * g.H;
            float* Or = Lout + img * st.out + (size_t)y * g.P;
            const int nfull = n >> 2;
            for (int v = tid; v < nfull; v += blockDim.x) {
                const float4 u = reinterpret_cast<const float4*>(sU)[v];
                const float4 x = reinterpret_cast<const float4*>(sL)[v];
                reinterpret_cast<float4*>(Or)[v] =
                    make_float4(0.5f * (u.x + x.x), 0.5f * (u.y + x.y), 0.5f * (u.z + x.z), 0.5f * (u.w + x.w));
            }
            for (int j = 4 * nfull + tid; j < n; j += blockDim.x) Or[j] = 0.5f * (sU[j] + sL[j]);
        }
        fence_proxy_async();  // generic-proxy writes of this stage before the TMA refills it
        __syncthreads();
    }
}

// -------------------------------------------------------------------------------------------------------------
// Row systems, one WARP per row (the row pass runs first and writes V; the column pass then forms ½(U + V)).
// The row (L and c) is staged in shared memory; lane l owns the chunk [l·M, l·M + m) with M odd, so the lanes'
// strided sweeps hit 32 distinct banks.  The sweeps keep their coefficients in shared memory, in place:
// δ overwrites L, γ overwrites c (each c is read before its slot is reused), α goes to a third array.  The
// reduced system of one unknown per lane is solved by PCR over shuffles — no block barriers at all.
// Shared memory per warp: 3 row buffers.
constexpr int kRowWarps = 4;

__global__ void __launch_bounds__(32 * kRowWarps) k_aos_rows_warp(const float* __restrict__ L,
                                                                  const float* __restrict__ c, float* __restrict__ V,
                                                                  Strides st, Geom g, float tau, int M, int T,
                                                                  int total_rows) {
    extern __shared__ __align__(16) float rsm[];
    __shared__ __align__(8) uint64_t wbar[kRowWarps];
    const int n = g.W;
    const int Wp = (n + 3) & ~3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sL = rsm + warp * 3 * Wp;
    float* sC = sL + Wp;
    float* sA = sC + Wp;
    if (lane == 0) {
        mbar_init(&wbar[warp], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;
    const int j0 = lane * M;
    const int m = lane < T ? ((lane == T - 1) ? n - j0 : M) : 0;
    const bool first = lane == 0, last = lane == T - 1;
    for (int q = blockIdx.x * kRowWarps + warp; q < total_rows; q += gridDim.x * kRowWarps) {
        const int img = q / g.H, y = q - img * g.H;
        const size_t ry = (size_t)y * g.P;
        if (lane == 0) {  // the TMA engine streams the row's L and c into this warp's buffers
            fence_proxy_async();
            mbar_arrive_expect_tx(&wbar[warp], 8u * (uint32_t)Wp);
            bulk_g2s(sL, L + img * st.L + ry, 4u * (uint32_t)Wp, &wbar[warp]);
            bulk_g2s(sC, c + img * st.c + ry, 4u * (uint32_t)Wp, &wbar[warp]);
        }
        mbar_wait(&wbar[warp], phase);
        phase ^= 1u;
        float A = 0.f, C = 0.f, D = 0.f, lA = 0.f, lG = 0.f, lD = 0.f;
        if (m > 0) {
            const float cprev = first ? 0.f : sC[j0 - 1];
            const float cnext = last ? 0.f : sC[j0 + m];
            const float c0 = sC[j0], c1 = sC[j0 + 1], d0 = sL[j0];
            __syncwarp(0xffffffffu >> (32 - T));  // neighbour boundary values read before any slot is reused
            // downward sweep, rows 1..m-1 (virtual row 0: α = -1, γ = 0, δ = 0); q_i = τ(c_{i-1} + c_i)
            float pa = -1.f, pg = 0.f, pd = 0.f;
            float cm = c0, cc = c1;
            float tqi = tau * (c0 + c1);  // τ(c_0 + c_1) = a_1 magnitude
#pragma unroll 4
            for (int i = 1; i < m; ++i) {
                const float cn = (i + 1 < m) ? sC[j0 + i + 1] : cnext;
                const float tqn = (i == m - 1 && last) ? 0.f : tau * (cc + cn);
                const float r = frcp(1.f + tqi + tqn + tqi * pg);
                const float na = tqi * pa * r;
                const float ng = -tqn * r;
                const float nd = fmaf(tqi, pd, sL[j0 + i]) * r;
                sA[j0 + i] = na;
                sC[j0 + i] = ng;  // c_i was consumed into cc / tqi
                sL[j0 + i] = nd;
                pa = na;
                pg = ng;
                pd = nd;
                cm = cc;
                cc = cn;
                tqi = tqn;
            }
            (void)cm;
            lA = pa;
            lG = pg;
            lD = pd;
            // upward sweep, rows m-2..1 (virtual row m-1: α' = 0, γ' = -1, δ' = 0)
            float na = 0.f, ng = -1.f, nd = 0.f;
#pragma unroll 4
            for (int i = m - 2; i >= 1; --i) {
                const float gi = sC[j0 + i];
                const float a2 = sA[j0 + i] - gi * na;
                const float g2 = -gi * ng;
                const float d2 = sL[j0 + i] - gi * nd;
                sA[j0 + i] = a2;
                sC[j0 + i] = g2;
                sL[j0 + i] = d2;
                na = a2;
                ng = g2;
                nd = d2;
            }
            // row 0: a0 = -τ(c_{-1} + c_0) (0 on the first chunk), cc0 = -τ(c_0 + c_1)
            const float tq0 = first ? 0.f : tau * (cprev + c0);
            const float tq1 = tau * (c0 + c1);
            const float rB = frcp(fmaf(tq1, na, 1.f + tq0 + tq1));
            A = -tq0 * rB;
            C = tq1 * ng * rB;
            D = fmaf(tq1, nd, d0) * rB;
        }
        // reduced system in the lanes' first unknowns f_l (identity rows for idle lanes)
        const float pAl = __shfl_up_sync(0xffffffffu, lA, 1), pGl = __shfl_up_sync(0xffffffffu, lG, 1);
        const float pDl = __shfl_up_sync(0xffffffffu, lD, 1);
        float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
        if (m > 0) {
            const float qa = first ? 0.f : pAl, qg = first ? 0.f : pGl, qd = first ? 0.f : pDl;
            af = -A * qa;
            bf = 1.f - A * qg - C * lA;
            cf = -C * lG;
            df = D - A * qd - C * lD;
        }
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
            const bool hm = lane >= s2, hp = lane + s2 < 32;
            const float am = __shfl_up_sync(0xffffffffu, af, s2), bm = __shfl_up_sync(0xffffffffu, bf, s2);
            const float cmm = __shfl_up_sync(0xffffffffu, cf, s2), dm = __shfl_up_sync(0xffffffffu, df, s2);
            const float ap = __shfl_down_sync(0xffffffffu, af, s2), bp = __shfl_down_sync(0xffffffffu, bf, s2);
            const float cp = __shfl_down_sync(0xffffffffu, cf, s2), dp = __shfl_down_sync(0xffffffffu, df, s2);
            const float k1 = hm ? af * frcp(bm) : 0.f;
            const float k2 = hp ? cf * frcp(bp) : 0.f;
            af = hm ? -am * k1 : 0.f;
            cf = hp ? -cp * k2 : 0.f;
            bf = bf - (hm ? cmm * k1 : 0.f) - (hp ? ap * k2 : 0.f);
            df = df - (hm ? dm * k1 : 0.f) - (hp ? dp * k2 : 0.f);
        }
        const float xf = df * frcp(bf);
        const float xnext = __shfl_down_sync(0xffffffffu, xf, 1);
        if (m > 0) {
            const float xl = lD - lA * xf - lG * (last ? 0.f : xnext);
#pragma unroll 4
            for (int i = 1; i < m - 1; ++i) sL[j0 + i] = sL[j0 + i] - sA[j0 + i] * xf - sC[j0 + i] * xl;
            sL[j0] = xf;
            sL[j0 + m - 1] = xl;
        }
        __syncwarp();
        float4* Vr = reinterpret_cast<float4*>(V + img * st.out + ry);
        for (int v = lane; v < (Wp >> 2); v += 32) Vr[v] = reinterpret_cast<const float4*>(sL)[v];
        fence_proxy_async();  // generic reads/writes of the buffers before the next TMA refill
        __syncwarp();
    }
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

template <int CW, int M, int NT>
void run_cols(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg, float tau,
              cudaStream_t s) {
    const int T = n_chunks(g.H, M);
    const int TP = round_up(T, 32 / CW);
    const size_t smem = sizeof(float) * 7 * CW * TP;
    dim3 grid((g.W + CW - 1) / CW, 1, nimg);
    k_aos_cols<CW, M, NT><<<grid, CW * TP, smem, s>>>(L, c, U, Lout, st, g, tau, T, TP);
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int M>
void run_rows(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg, float tau,
              cudaStream_t s) {
    const int T = n_chunks(g.W, M);
    const int TP = round_up(T, 32);
    const int Wp = (g.W + 3) & ~3;
    const size_t smem = sizeof(float) * (6 * Wp + 4 * (TP + 1) + 64 + 3 * TP + 4) + 2 * sizeof(uint64_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_aos_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const int total = g.H * nimg;
    int per_sm = (int)((220 * 1024) / (smem + 1024));
    per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
    const int grid = total < num_sms() * per_sm ? total : num_sms() * per_sm;
    k_aos_rows<M><<<grid, TP, smem, s>>>(L, c, U, Lout, st, g, tau, T, TP, total);
}

}  // namespace

// Column chunk length: T = n_chunks(H, M) must fit the CTA (CW*TP <= NT).
bool launch_aos_cols(const float* L, const float* c, const float* V, float* Lout, Strides st, Geom g, int nimg,
                     float tau, cudaStream_t s) {
    const int H = g.H;
    if (H <= 128 * 4) run_cols<8, 4, 1024>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 128 * 6) run_cols<8, 6, 1024>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 128 * 8) run_cols<8, 8, 1024>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 128 * 10) run_cols<8, 10, 1024>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 128 * 12) run_cols<8, 12, 1024>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 256 * 16) run_cols<2, 16, 512>(L, c, V, Lout, st, g, nimg, tau, s);
    else if (H <= 256 * 32) run_cols<2, 32, 512>(L, c, V, Lout, st, g, nimg, tau, s);
    else return false;
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
