// aos.cu — semi-implicit AOS step of Eq. 4 (readings A1, A2) on sm_100a.
//
// L_i = ½[(I − 2τA_x(c))⁻¹ + (I − 2τA_y(c))⁻¹] L_{i−1}: H row systems of length W (k_aos_rows_cta → V, first) and
// W column systems of length H (k_aos_cols → L_i = ½(U + V), second).  Every line is tridiagonal with
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
//   columns: a CTA owns CW adjacent columns; a warp covers CW columns × 32/CW chunks, so every global request is
//            whole 32-byte sectors; the reduced systems are solved by PCR in shared memory; V is prefetched with
//            cp.async behind the solve and L_i = ½(U + V) is written directly.
//            (Measured alternatives, all slower on B200 for 1920x1200: TMA-pipelined persistent strips 80 ms,
//            three register-light passes 88 ms, re-mapped warp SPIKE 77 ms, vs 66 ms per 256-image step here.)
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
    float* sv = sld + NTOT;  // V chunk, prefetched with cp.async while the solve runs: [MC][NTOT]
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int x = blockIdx.x * CW + cx;
    const bool active = (p < T) && (x < g.W);
    const int n = g.H;
    const int j0 = p * M;
    const int j1 = (p == T - 1) ? n : j0 + M;
    const int m = active ? j1 - j0 : 0;

    Chunk<MC> ch;
    if (active) {  // the V chunk streams into shared memory behind the solve
        const float* Vg = U + blockIdx.z * st.U + (size_t)j0 * g.P + x;
#pragma unroll
        for (int i = 0; i < MC; ++i)
            if (i < m) cp_async4(sv + i * NTOT + threadIdx.x, Vg + (size_t)i * g.P);
    }
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
    // L_i = ½(U + V): the row pass already wrote V (prefetched into sv); the average is formed here.
    cp_async_wait_all();
    const float* vv = sv + threadIdx.x;
    float* Oc = Lout + blockIdx.z * st.out + (size_t)j0 * g.P + x;
    Oc[0] = 0.5f * (xf + vv[0]);
#pragma unroll
    for (int i = 1; i < MC; ++i) {
        if (i < m - 1) Oc[(size_t)i * g.P] = 0.5f * (ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl + vv[i * NTOT]);
    }
    Oc[(size_t)(m - 1) * g.P] = 0.5f * (xl + vv[(m - 1) * NTOT]);
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
    const size_t smem = sizeof(float) * (7 + M + 1) * CW * TP;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_aos_cols<CW, M, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid((g.W + CW - 1) / CW, 1, nimg);
    k_aos_cols<CW, M, NT><<<grid, CW * TP, smem, s>>>(L, c, U, Lout, st, g, tau, T, TP);
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
