// aos.cu — semi-implicit AOS step of Eq. 4 (readings A1, A2) on sm_100a.
//
// L_i = ½[(I − 2τA_y(c))⁻¹ + (I − 2τA_x(c))⁻¹] L_{i−1}: W column systems of length H (k_aos_cols → U) and
// H row systems of length W (k_aos_rows → L_i = ½(U + V)).  Every line is tridiagonal with
//   a_j = −τ(c_{j−1} + c_j),  cc_j = −τ(c_j + c_{j+1}),  b_j = 1 − a_j − cc_j   (Neumann ends: a_0 = cc_{n−1} = 0).
//
// Parallel scheme (partition / "Thomas–PCR hybrid"): a line of n samples is cut into T chunks of
// m ≤ M samples, one thread per chunk.  Each thread
//   1. eliminates its chunk in registers (downward sweep keeping x_first, then upward sweep keeping x_last), so
//      every interior sample reads x_i = δ'_i − α'_i x_first − γ'_i x_last, and the chunk contributes two
//      reduced equations: F_p: A x_{last,p−1} + x_{first,p} + C x_{last,p} = D,
//                         L_p: α x_{first,p} + x_{last,p} + γ x_{first,p+1} = δ;
//   2. substitutes L_{p−1}, L_p into F_p → a tridiagonal system in the T unknowns x_{first,p}, solved by parallel
//      cyclic reduction in shared memory (log2 T steps);
//   3. evaluates its samples from the two chunk-end values.
// Column lines are read straight from global memory (a warp covers CW adjacent columns × 32/CW chunks: every
// request is whole 32-byte sectors).  Row lines are staged through shared memory with coalesced loads; each
// chunk starts at an odd word stride so the per-thread sweeps are bank-conflict free.
#include "kaze_internal.cuh"

namespace kz {

namespace {

// Solve the reduced system of T "first" unknowns held one per thread (p = chunk index, s = system index within
// the CTA).  eq: (af, bf, cf, df).  Returns x_first of this chunk.  Threads with p >= T carry identity rows.
// sa..sd: shared arrays [NS][TP] (TP = padded chunk count, power of two not required).
__device__ __forceinline__ float pcr_solve(float af, float bf, float cf, float df, int p, int TP, float* sa,
                                           float* sb, float* sc, float* sd, int idx /* s*TP + p */) {
    for (int st = 1; st < TP; st <<= 1) {
        sa[idx] = af;
        sb[idx] = bf;
        sc[idx] = cf;
        sd[idx] = df;
        __syncthreads();
        float na = 0.f, nc = 0.f, nb = bf, nd = df;
        if (p - st >= 0) {
            float k1 = af / sb[idx - st];
            na = -sa[idx - st] * k1;
            nb -= sc[idx - st] * k1;
            nd -= sd[idx - st] * k1;
        }
        if (p + st < TP) {
            float k2 = cf / sb[idx + st];
            nc = -sc[idx + st] * k2;
            nb -= sa[idx + st] * k2;
            nd -= sd[idx + st] * k2;
        }
        __syncthreads();
        af = na;
        bf = nb;
        cf = nc;
        df = nd;
    }
    return df / bf;
}

// Per-thread chunk elimination on registers.  Inputs through the loader functor ld(i) → (d_i, c_{j-1}, c_j,
// c_{j+1} flags).  We pass the line-local sample values explicitly to keep the code shared by both passes.
template <int M>
struct Chunk {
    float al[M], ga[M], de[M];  // α', γ', δ' for i = 1..m-2 (index i), forward values before the upward sweep
    float A, C, D;              // first equation (normalised)
    float lA, lG, lD;           // last equation  α x_first + x_last + γ x_next_first = δ
};

// cprev = c at sample j0-1 (ignored if j0 == 0), cv[i] = c at j0+i, cnext = c at j0+m (ignored if j0+m == n).
template <int M>
__device__ __forceinline__ void eliminate(Chunk<M>& ch, const float (&dv)[M], const float (&cv)[M], float cprev,
                                          float cnext, int m, bool first_chunk, bool last_chunk, float tau) {
    // coefficients of row i: a_i, b_i, cc_i
    auto coef = [&](int i, float& a, float& b, float& cc) {
        float cl = (i == 0) ? cprev : cv[i - 1 < 0 ? 0 : i - 1];
        float cm = cv[i];
        float cr = (i == m - 1) ? cnext : cv[i + 1 < M ? i + 1 : M - 1];
        a = (i == 0 && first_chunk) ? 0.f : -tau * (cl + cm);
        cc = (i == m - 1 && last_chunk) ? 0.f : -tau * (cm + cr);
        b = 1.f - a - cc;
    };
    // downward sweep (rows 1..m-1), virtual row 0: α = -1, γ = 0, δ = 0
    float pa = -1.f, pg = 0.f, pd = 0.f;
#pragma unroll
    for (int i = 1; i < M; ++i) {
        if (i < m) {
            float a, b, cc;
            coef(i, a, b, cc);
            float r = 1.f / (b - a * pg);
            float na = -a * pa * r;
            float ng = cc * r;
            float nd = (dv[i] - a * pd) * r;
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
    for (int i = M - 2; i >= 1; --i) {
        if (i <= m - 2) {
            float g = ch.ga[i];
            float a2 = ch.al[i] - g * na;
            float g2 = -g * ng;
            float d2 = ch.de[i] - g * nd;
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
    float B = b0 - c0 * na;
    float rB = 1.f / B;
    ch.A = a0 * rB;
    ch.C = -c0 * ng * rB;
    ch.D = (dv[0] - c0 * nd) * rB;
}

// -------------------------------------------------------------------------------------------------------------
// Column systems.  Thread (cx, p): column x0 + cx, chunk p of T.  blockDim.x = CW * TP.
template <int CW, int M, int NT>
__global__ void __launch_bounds__(NT) k_aos_cols(const float* __restrict__ L, const float* __restrict__ c,
                                                 float* __restrict__ U, Strides st, Geom g, float tau, int T, int TP) {
    extern __shared__ float sm[];
    const int NS = CW;
    float* sa = sm;
    float* sb = sa + NS * TP;
    float* sc = sb + NS * TP;
    float* sd = sc + NS * TP;
    float* sla = sd + NS * TP;  // last-equation exchange
    float* slg = sla + NS * TP;
    float* sld = slg + NS * TP;
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int x = blockIdx.x * CW + cx;
    const bool active = (p < T) && (x < g.W);
    const int n = g.H;
    const int j0 = (int)(((long long)p * n) / T), j1 = (int)(((long long)(p + 1) * n) / T);
    const int m = active ? j1 - j0 : 0;

    Chunk<M> ch;
    if (active) {
        float dv[M], cv[M];
        const float* Lc = L + blockIdx.z * st.L + x;
        const float* cc = c + blockIdx.z * st.c + x;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            if (i < m) {
                dv[i] = __ldg(Lc + (size_t)(j0 + i) * g.P);
                cv[i] = __ldg(cc + (size_t)(j0 + i) * g.P);
            } else {
                dv[i] = 0.f;
                cv[i] = 0.f;
            }
        }
        float cprev = j0 > 0 ? __ldg(cc + (size_t)(j0 - 1) * g.P) : 0.f;
        float cnext = j1 < n ? __ldg(cc + (size_t)j1 * g.P) : 0.f;
        eliminate<M>(ch, dv, cv, cprev, cnext, m, j0 == 0, j1 == n, tau);
    } else {
        ch.A = ch.C = ch.D = 0.f;
        ch.lA = ch.lG = ch.lD = 0.f;
    }
    const int idx = cx * TP + p;
    sla[idx] = ch.lA;
    slg[idx] = ch.lG;
    sld[idx] = ch.lD;
    __syncthreads();
    float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
    if (active) {
        float pA = 0.f, pG = 0.f, pD = 0.f;
        if (p > 0) {
            pA = sla[idx - 1];
            pG = slg[idx - 1];
            pD = sld[idx - 1];
        }
        af = -ch.A * pA;
        bf = 1.f - ch.A * pG - ch.C * ch.lA;
        cf = -ch.C * ch.lG;
        df = ch.D - ch.A * pD - ch.C * ch.lD;
    }
    float xf = pcr_solve(af, bf, cf, df, p, TP, sa, sb, sc, sd, idx);
    sa[idx] = xf;
    __syncthreads();
    if (!active) return;
    float xnext = (p + 1 < T) ? sa[idx + 1] : 0.f;
    float xl = ch.lD - ch.lA * xf - ch.lG * xnext;
    float* Uc = U + blockIdx.z * st.U + x;
    Uc[(size_t)j0 * g.P] = xf;
#pragma unroll
    for (int i = 1; i < M; ++i) {
        if (i < m - 1) Uc[(size_t)(j0 + i) * g.P] = ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl;
    }
    Uc[(size_t)(j1 - 1) * g.P] = xl;
}

// -------------------------------------------------------------------------------------------------------------
// Row systems: one row per CTA, staged in shared memory (chunk p at word offset p*S, S odd).
template <int M>
__global__ void __launch_bounds__(256) k_aos_rows(const float* __restrict__ L, const float* __restrict__ c,
                                                  const float* __restrict__ U, float* __restrict__ Lout, Strides st,
                                                  Geom g, float tau, int T, int TP) {
    extern __shared__ float sm[];
    constexpr int S = (M % 2 == 1) ? M : M + 1;
    float* sL = sm;                // T*S
    float* sC = sL + TP * S;       // T*S
    float* sa = sC + TP * S;       // TP each
    float* sb = sa + TP;
    float* sc = sb + TP;
    float* sd = sc + TP;
    float* sla = sd + TP;
    float* slg = sla + TP;
    float* sld = slg + TP;
    const int n = g.W;
    const int y = blockIdx.x;
    const size_t ry = (size_t)y * g.P;
    const float* Lr = L + blockIdx.z * st.L + ry;
    const float* cr = c + blockIdx.z * st.c + ry;
    const float* Ur = U + blockIdx.z * st.U + ry;
    float* Or = Lout + blockIdx.z * st.out + ry;
    // stage the row: sample j lives in chunk p(j) = floor(((j+1)T - 1)/n) at offset j - start(p)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        int pj = (int)((((long long)(j + 1)) * T - 1) / n);
        int s0 = (int)(((long long)pj * n) / T);
        sL[pj * S + (j - s0)] = __ldg(Lr + j);
        sC[pj * S + (j - s0)] = __ldg(cr + j);
    }
    __syncthreads();
    const int p = threadIdx.x;
    const bool active = p < T;
    const int j0 = (int)(((long long)p * n) / T), j1 = (int)(((long long)(p + 1) * n) / T);
    const int m = active ? j1 - j0 : 0;
    Chunk<M> ch;
    if (active) {
        float dv[M], cv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            dv[i] = i < m ? sL[p * S + i] : 0.f;
            cv[i] = i < m ? sC[p * S + i] : 0.f;
        }
        float cprev = 0.f, cnext = 0.f;
        if (p > 0) {
            int mp = j0 - (int)(((long long)(p - 1) * n) / T);
            cprev = sC[(p - 1) * S + mp - 1];
        }
        if (p + 1 < T) cnext = sC[(p + 1) * S];
        eliminate<M>(ch, dv, cv, cprev, cnext, m, p == 0, p == T - 1, tau);
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
    float xf = pcr_solve(af, bf, cf, df, p, TP, sa, sb, sc, sd, p);
    sa[p] = xf;
    __syncthreads();
    if (active) {
        float xnext = (p + 1 < T) ? sa[p + 1] : 0.f;
        float xl = ch.lD - ch.lA * xf - ch.lG * xnext;
        sL[p * S] = xf;
#pragma unroll
        for (int i = 1; i < M; ++i)
            if (i < m - 1) sL[p * S + i] = ch.de[i] - ch.al[i] * xf - ch.ga[i] * xl;
        sL[p * S + m - 1] = xl;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        int pj = (int)((((long long)(j + 1)) * T - 1) / n);
        int s0 = (int)(((long long)pj * n) / T);
        Or[j] = 0.5f * (__ldg(Ur + j) + sL[pj * S + (j - s0)]);
    }
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

template <int CW, int M, int NT>
void run_cols(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau, cudaStream_t s) {
    int T = (g.H + M - 1) / M;
    int TP = round_up(T, 32 / CW);
    int threads = CW * TP;
    size_t smem = sizeof(float) * 7 * CW * TP;
    dim3 grid((g.W + CW - 1) / CW, 1, nimg);
    k_aos_cols<CW, M, NT><<<grid, threads, smem, s>>>(L, c, U, st, g, tau, T, TP);
}

template <int M>
void run_rows(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg, float tau,
              cudaStream_t s) {
    constexpr int S = (M % 2 == 1) ? M : M + 1;
    int T = (g.W + M - 1) / M;
    int TP = round_up(T, 32);
    size_t smem = sizeof(float) * (2 * TP * S + 7 * TP);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_aos_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(g.H, 1, nimg);
    k_aos_rows<M><<<grid, TP, smem, s>>>(L, c, U, Lout, st, g, tau, T, TP);
}

}  // namespace

// Line length n → chunk length M: the smallest instantiated M >= 4 that keeps T = ceil(n/M) within the CTA.
// (M >= 4 keeps every balanced chunk at >= 2 samples for n >= 32.)
bool launch_aos_cols(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau,
                     cudaStream_t s) {
    const int H = g.H;
    if (H <= 128 * 4) run_cols<8, 4, 1024>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 128 * 6) run_cols<8, 6, 1024>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 128 * 8) run_cols<8, 8, 1024>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 128 * 10) run_cols<8, 10, 1024>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 128 * 12) run_cols<8, 12, 1024>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 256 * 16) run_cols<2, 16, 512>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 256 * 32) run_cols<2, 32, 512>(L, c, U, st, g, nimg, tau, s);
    else return false;
    return true;
}

bool launch_aos_rows(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg,
                     float tau, cudaStream_t s) {
    const int W = g.W;
    if (W <= 256 * 4) run_rows<4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 8) run_rows<8>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 16) run_rows<16>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 32) run_rows<32>(L, c, U, Lout, st, g, nimg, tau, s);
    else return false;
    return true;
}

}  // namespace kz
