// aos.cu — semi-implicit AOS step of Eq. 4 (readings A1, A2) on sm_100a.
//
// L_i = ½[(I − 2τA_y(c))⁻¹ + (I − 2τA_x(c))⁻¹] L_{i−1}: W column systems of length H (k_aos_cols_u → U, first
// pass, 12 B/px) and H row systems of length W (k_aos_rows_cta → L_i = ½(U + V), second pass, 16 B/px).  Every
// line is tridiagonal with
//   a_j = −τ(c_{j−1} + c_j),  cc_j = −τ(c_j + c_{j+1}),  b_j = 1 − a_j − cc_j   (Neumann ends: a_0 = cc_{n−1} = 0).
//
// Both passes use the partition ("Thomas–PCR hybrid") scheme of DESIGN.md §6: a line is cut into T chunks of M
// samples, one thread per chunk.  Each thread eliminates its chunk in registers, leaving two reduced equations
// (its first sample in terms of the previous chunk's last, its last in terms of the next chunk's first);
// substituting the neighbour's last equation gives a tridiagonal system in the T chunk-first unknowns; after it
// is solved every thread evaluates its samples.
//   columns: a CTA owns CW adjacent columns; a warp covers CW columns × 32/CW chunks, so every global request is
//            whole 32-byte sectors.  Register-light elimination (independent down and up sweeps, then a Dirichlet
//            Thomas sweep in place: two live values per sample) lets two 480-thread CTAs share an SM, so one
//            CTA's loads overlap the other's solve; the reduced systems are solved by PCR in shared memory.
//            The ragged last chunk is padded with decoupled rows (zero edge weights), so there is one path.
//            Columns run first because the row pass reads a third array almost for free: its TMA bulk copies
//            stream L, c and U, and it writes L_i = ½(U + V) with 16-byte stores.  (Measured on B200, 256-image
//            1920x1200 step: this order and kernel 34.7 + 25.0 ms vs 58.3 + 22.9 ms for rows-first with a
//            three-value column kernel; earlier column variants — TMA-pipelined persistent strips, three
//            register-light passes, re-mapped warp SPIKE — were slower still.  Two columns per thread in packed
//            fp32x2 (FFMA2/FMUL2, M = 10 to fit 64 registers) issued 35 instead of 55 instructions per pixel but
//            ran 42.0 vs 32.2 ms: twice the chunks make the shared-memory PCR (7 steps, float2) the bottleneck.
//            CTA shape at M = 20: 4 columns x 4 CTAs/SM 39.3 ms, 16 columns x 1 CTA/SM 34.1, 8 x 2 (kept) 29.5.)
//            Default for H <= 64·19 (round 2): k_aos_cols_tmap — persistent CTAs, one per SM, double-buffered TMA
//            strips, and the reduced systems solved by one warp per column with a shuffle PCR (3 CTA barriers per
//            strip): 24.3 vs 27.4 ms for the per-strip TMA kernel k_aos_cols_tma (kept for KAZE_COLS_PERSIST=0),
//            k_aos_cols_u for taller images.
//   rows:    one CTA (4 or 8 warps) per row.  The TMA engine streams the row's L, c and U into shared memory (1-D
//            bulk copies, mbarrier), M is odd so the strided chunk reads are conflict free; the reduced system is
//            solved by a warp-level SPIKE (shuffle PCR on three right-hand sides + a 2·NW-unknown boundary solve).
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kaze_internal.cuh"
#include "ptx.cuh"

namespace kz {

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {  // thread-safe one-time lookup
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}
}  // namespace

bool encode_f32_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                    const cuuint32_t* box) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

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

// Warp PCR for the column pass: the reduced system of one column (64 chunk unknowns, identity rows past the real
// ones) solved by ONE warp, two unknowns per lane (slots r = 2·lane, 2·lane + 1), all levels by shuffles — no CTA
// barriers (the shared-memory PCR above takes two per level, twelve at 64 chunks).  In: the lane's two rows
// (a, b, c, d); returns x of its two slots.
__device__ __forceinline__ float2 warp_pcr64(float (&a)[2], float (&b)[2], float (&c)[2], float (&d)[2], int lane) {
#pragma unroll
    for (int st = 1; st < 64; st <<= 1) {
        float na[2], nb[2], nc[2], nd[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int r = 2 * lane + s, jm = r - st, jp = r + st;
            const bool hm = jm >= 0, hp = jp < 64;
            const int sm_ = (s - st) & 1, sp_ = (s + st) & 1;  // slots of the partners (uniform)
            const int lm = hm ? jm >> 1 : 0, lp = hp ? jp >> 1 : 0;
            const float am = __shfl_sync(0xffffffffu, sm_ ? a[1] : a[0], lm);
            const float bm = __shfl_sync(0xffffffffu, sm_ ? b[1] : b[0], lm);
            const float cm = __shfl_sync(0xffffffffu, sm_ ? c[1] : c[0], lm);
            const float dm = __shfl_sync(0xffffffffu, sm_ ? d[1] : d[0], lm);
            const float ap = __shfl_sync(0xffffffffu, sp_ ? a[1] : a[0], lp);
            const float bp = __shfl_sync(0xffffffffu, sp_ ? b[1] : b[0], lp);
            const float cp = __shfl_sync(0xffffffffu, sp_ ? c[1] : c[0], lp);
            const float dp = __shfl_sync(0xffffffffu, sp_ ? d[1] : d[0], lp);
            const float k1 = hm ? a[s] * frcp(bm) : 0.f;
            const float k2 = hp ? c[s] * frcp(bp) : 0.f;
            na[s] = -am * k1;
            nc[s] = -cp * k2;
            nb[s] = b[s] - cm * k1 - ap * k2;
            nd[s] = d[s] - dm * k1 - dp * k2;
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            a[s] = na[s];
            b[s] = nb[s];
            c[s] = nc[s];
            d[s] = nd[s];
        }
    }
    return make_float2(d[0] * frcp(b[0]), d[1] * frcp(b[1]));
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

// -------------------------------------------------------------------------------------------------------------
// Column systems (first pass: U = column solves).  Thread (cx, p): column x0 + cx, chunk p of T; blockDim.x =
// CW * TP, shared index p*CW + cx.  A warp covers CW adjacent columns x 32/CW chunks (whole 32-byte sectors).
//
// Register-light elimination (two values per sample stay live instead of three): with the chunk's samples
// x_0..x_{m-1}, edge weights tq_i = τ(c_{i-1} + c_i) (a_i = −tq_i, cc_i = −tq_{i+1}, b_i = 1 + tq_i + tq_{i+1}),
//   down sweep, x_0 symbolic:        x_{m-1} = F − G·x_m − Hh·x_0          (the chunk's "last equation")
//   up sweep, x_{m-1} symbolic:      x_0 + A·x_{−1} + C·x_{m-1} = D        (its "first equation")
// Both sweeps read only (L, tq) and keep O(1) state.  Substituting the neighbours' last equations gives a
// tridiagonal system in the chunk-first unknowns X_k (PCR in shared memory); x_{m-1} follows from the last
// equation, and the interior is a Dirichlet problem solved by a Thomas sweep that overwrites (L, tq) in place.
struct ChunkEq {
    float A, C, D;     // first equation
    float lF, lG, lH;  // last equation
};

// Every chunk has exactly M samples: samples past the line end are padding rows decoupled by zero edge weights
// (b = 1, d = 0), so one branch-free path serves the ragged last chunk too.
template <int M>
__device__ __forceinline__ void chunk_reduce(const float (&dv)[M], const float (&tq)[M + 1], ChunkEq& e) {
    float F = 0.f, G = 0.f, Hh = -1.f;
#pragma unroll
    for (int i = 1; i < M; ++i) {
        const float r = frcp(fmaf(tq[i], G, 1.f + tq[i] + tq[i + 1]));  // b_i − a_i G
        F = fmaf(tq[i], F, dv[i]) * r;
        Hh = tq[i] * Hh * r;
        G = -tq[i + 1] * r;
    }
    e.lF = F;
    e.lG = G;
    e.lH = Hh;
    float P = 0.f, Q = 0.f, S = -1.f;
#pragma unroll
    for (int i = M - 2; i >= 1; --i) {
        const float r = frcp(fmaf(tq[i + 1], Q, 1.f + tq[i] + tq[i + 1]));  // b_i − cc_i Q
        P = fmaf(tq[i + 1], P, dv[i]) * r;
        S = tq[i + 1] * S * r;
        Q = -tq[i] * r;
    }
    const float rB = frcp(fmaf(tq[1], Q, 1.f + tq[0] + tq[1]));
    e.A = -tq[0] * rB;
    e.C = tq[1] * S * rB;
    e.D = fmaf(tq[1], P, dv[0]) * rB;
}

// Interior of the chunk with x_0 = x0 and x_{M-1} = xl known; writes the samples j0+i < n at out + o0 + i·P (32-bit
// element offsets from an opaque base: one IMAD.WIDE per address).  FULL: every sample is inside the line.
template <int M, bool FULL>
__device__ __forceinline__ void chunk_finish(float (&dv)[M], float (&tq)[M + 1], float x0, float xl,
                                             float* __restrict__ out, unsigned o0, unsigned P, int nvalid) {
    float Fp = x0, G = 0.f;
#pragma unroll
    for (int i = 1; i < M - 1; ++i) {
        const float r = frcp(fmaf(tq[i], G, 1.f + tq[i] + tq[i + 1]));
        Fp = fmaf(tq[i], Fp, dv[i]) * r;
        G = -tq[i + 1] * r;
        dv[i] = Fp;  // F'_i
        tq[i] = G;   // G_i
    }
    __stwb(out + o0, x0);  // st.global (the opaque base hides the address space)
    if (FULL || M - 1 < nvalid) __stwb(out + (o0 + (M - 1) * P), xl);
    float xn = xl;
#pragma unroll
    for (int i = M - 2; i >= 1; --i) {
        xn = fmaf(-tq[i], xn, dv[i]);
        if (FULL || i < nvalid) __stwb(out + (o0 + i * P), xn);
    }
}

template <int CW, int M, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_aos_cols_u(const float* __restrict__ L, const float* __restrict__ c,
                                                         float* __restrict__ U, Strides st, Geom g, float tau, int T,
                                                         int TP) {
    KZ_PDL_PROLOGUE();
    extern __shared__ float sm[];
    const int NTOT = CW * TP;
    float* sa = sm;
    float* sb = sa + NTOT;
    float* sc = sb + NTOT;
    float* sd = sc + NTOT;
    float* slF = sd + NTOT;  // last-equation exchange
    float* slG = slF + NTOT;
    float* slH = slG + NTOT;
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int x = blockIdx.x * CW + cx;
    const bool active = (p < T) && (x < g.W);
    const int n = g.H;
    const int j0 = p * M;
    const int nvalid = n - j0;  // samples of this chunk inside the line (>= 1 for p < T)
    float dv[M], tq[M + 1];
    ChunkEq e{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // 32-bit element offsets from opaque per-image bases (the plane is < 2^32 elements)
    const int img = batch_image(blockIdx.z, gridDim.z, g);
    const float* Lb = opaque(L + img * st.L);
    const float* cb = opaque(c + img * st.c);
    const unsigned P = (unsigned)g.P, o0 = (unsigned)j0 * P + (unsigned)x;
    const bool full = nvalid > M;  // all M samples and the next chunk's first sample exist
    if (active) {
        float cv[M];
        float cprev = 0.f, cnext = 0.f;
        if (full) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                dv[i] = __ldg(Lb + (o0 + i * P));
                cv[i] = __ldg(cb + (o0 + i * P));
            }
            cnext = __ldg(cb + (o0 + M * P));
        } else {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const bool in = i < nvalid;
                dv[i] = in ? __ldg(Lb + (o0 + i * P)) : 0.f;
                cv[i] = in ? __ldg(cb + (o0 + i * P)) : 0.f;
            }
        }
        if (j0 > 0) cprev = __ldg(cb + (o0 - P));
        // edge i joins samples j0+i-1 and j0+i; it exists iff 1 <= j0+i <= n-1 (Neumann ends, padding decoupled)
        tq[0] = j0 > 0 ? tau * (cprev + cv[0]) : 0.f;
        if (full) {
#pragma unroll
            for (int i = 1; i < M; ++i) tq[i] = tau * (cv[i - 1] + cv[i]);
            tq[M] = tau * (cv[M - 1] + cnext);
        } else {
#pragma unroll
            for (int i = 1; i < M; ++i) tq[i] = i < nvalid ? tau * (cv[i - 1] + cv[i]) : 0.f;
            tq[M] = 0.f;
        }
        chunk_reduce<M>(dv, tq, e);
    }
    const int idx = p * CW + cx;
    slF[idx] = e.lF;
    slG[idx] = e.lG;
    slH[idx] = e.lH;
    __syncthreads();
    float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
    if (active) {
        float pF = 0.f, pG = 0.f, pH = 0.f;
        if (p > 0) {
            pF = slF[idx - CW];
            pG = slG[idx - CW];
            pH = slH[idx - CW];
        }
        // x_{-1} = pF − pG·X_k − pH·X_{k−1};  x_{M−1} = lF − lG·X_{k+1} − lH·X_k
        af = -e.A * pH;
        bf = 1.f - e.A * pG - e.C * e.lH;
        cf = -e.C * e.lG;
        df = e.D - e.A * pF - e.C * e.lF;
    }
    const float xf = pcr_solve(af, bf, cf, df, p, TP, CW, idx, sa, sb, sc, sd);
    sa[idx] = xf;
    __syncthreads();
    if (!active) return;
    const float xnext = (p + 1 < T) ? sa[idx + CW] : 0.f;
    const float xl = e.lF - e.lG * xnext - e.lH * xf;
    float* Ub = opaque(U + img * st.out);
    if (full) chunk_finish<M, true>(dv, tq, xf, xl, Ub, o0, P, nvalid);
    else chunk_finish<M, false>(dv, tq, xf, xl, Ub, o0, P, nvalid);
}

// Column pass with TMA-staged inputs (the default for H <= 64·19): one thread issues 3-D tiled tensor copies of the
// CTA's CW-column strip of L and c (boxes of CW x BR rows, zero fill past the image) into shared memory, [row][CW]
// floats, and every thread reads its chunk from there.  The chunk length M is odd, so the four chunks a warp covers
// (rows p·M + i, p = 4w..4w+3) fall in four different bank groups: one conflict-free LDS per sample and array
// instead of an LDG that touches four 32-byte sectors in four lines (41 such loads per thread kept the LSU/MIO queue
// full in the register-staged kernel above — mio_throttle was its top stall).  Solve and stores as above.
// chunk_finish into the CTA's shared staging rows (row stride CW) instead of global memory.
template <int M, bool FULL, int CW>
__device__ __forceinline__ void chunk_finish_smem(float (&dv)[M], float (&tq)[M + 1], float x0, float xl,
                                                  float* __restrict__ s, int nvalid) {
    float Fp = x0, G = 0.f;
#pragma unroll
    for (int i = 1; i < M - 1; ++i) {
        const float r = frcp(fmaf(tq[i], G, 1.f + tq[i] + tq[i + 1]));
        Fp = fmaf(tq[i], Fp, dv[i]) * r;
        G = -tq[i + 1] * r;
        dv[i] = Fp;
        tq[i] = G;
    }
    s[0] = x0;
    if (FULL || M - 1 < nvalid) s[(M - 1) * CW] = xl;
    float xn = xl;
#pragma unroll
    for (int i = M - 2; i >= 1; --i) {
        xn = fmaf(-tq[i], xn, dv[i]);
        if (FULL || i < nvalid) s[i * CW] = xn;
    }
}

template <int CW, int M, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_aos_cols_tma(const __grid_constant__ CUtensorMap tmL,
                                                           const __grid_constant__ CUtensorMap tmC,
                                                           const __grid_constant__ CUtensorMap tmU,
                                                           float* __restrict__ U, size_t u_stride, Geom g, float tau,
                                                           int T, int TP, int nbox, int BR) {
    KZ_PDL_PROLOGUE();
    extern __shared__ __align__(128) float smem_cols[];
    __shared__ __align__(8) uint64_t bar;
    const int HB = nbox * BR;
    float* smL = smem_cols;      // [HB][CW]
    float* smC = smL + HB * CW;  // [HB][CW]
    const int NTOT = CW * TP;
    float* sa = smC + HB * CW;
    float* sb = sa + NTOT;
    float* sc = sb + NTOT;
    float* sd = sc + NTOT;
    float* slF = sd + NTOT;
    float* slG = slF + NTOT;
    float* slH = slG + NTOT;
    const int x0 = blockIdx.x * CW, img = batch_image(blockIdx.z, gridDim.z, g);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 2u * (uint32_t)(HB * CW) * 4u);
        for (int b = 0; b < nbox; ++b) {
            tma_load_3d(smL + b * BR * CW, &tmL, x0, b * BR, img, &bar);
            tma_load_3d(smC + b * BR * CW, &tmC, x0, b * BR, img, &bar);
        }
    }
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int x = x0 + cx;
    const bool active = (p < T) && (x < g.W);
    const int n = g.H;
    const int j0 = p * M;
    const int nvalid = n - j0;
    float dv[M], tq[M + 1];
    ChunkEq e{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&bar, 0);
    if (active) {
        // padding samples of the last chunk (rows >= H; they may lie past the staged rows) read 0 and their edge
        // weights are zero, so they decouple exactly as in the register-staged kernel
        float cv[M];
        const bool full = nvalid > M;
        if (full) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                dv[i] = smL[(j0 + i) * CW + cx];
                cv[i] = smC[(j0 + i) * CW + cx];
            }
        } else {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                dv[i] = i < nvalid ? smL[(j0 + i) * CW + cx] : 0.f;
                cv[i] = i < nvalid ? smC[(j0 + i) * CW + cx] : 0.f;
            }
        }
        const float cprev = j0 > 0 ? smC[(j0 - 1) * CW + cx] : 0.f;
        tq[0] = j0 > 0 ? tau * (cprev + cv[0]) : 0.f;
        if (full) {
#pragma unroll
            for (int i = 1; i < M; ++i) tq[i] = tau * (cv[i - 1] + cv[i]);
            tq[M] = tau * (cv[M - 1] + smC[(j0 + M) * CW + cx]);
        } else {
#pragma unroll
            for (int i = 1; i < M; ++i) tq[i] = i < nvalid ? tau * (cv[i - 1] + cv[i]) : 0.f;
            tq[M] = 0.f;
        }
        chunk_reduce<M>(dv, tq, e);
    }
    const int idx = p * CW + cx;
    slF[idx] = e.lF;
    slG[idx] = e.lG;
    slH[idx] = e.lH;
    __syncthreads();
    float af = 0.f, bf = 1.f, cf = 0.f, df = 0.f;
    if (active) {
        float pF = 0.f, pG = 0.f, pH = 0.f;
        if (p > 0) {
            pF = slF[idx - CW];
            pG = slG[idx - CW];
            pH = slH[idx - CW];
        }
        af = -e.A * pH;
        bf = 1.f - e.A * pG - e.C * e.lH;
        cf = -e.C * e.lG;
        df = e.D - e.A * pF - e.C * e.lF;
    }
    const float xf = pcr_solve(af, bf, cf, df, p, TP, CW, idx, sa, sb, sc, sd);
    sa[idx] = xf;
    __syncthreads();
    // U goes to the L staging rows (every thread read its L samples before the first barrier) and leaves with one
    // tensor store per box: no per-sample global stores (19 STG touching four lines each per thread before)
    if (active) {
        const float xnext = (p + 1 < T) ? sa[idx + CW] : 0.f;
        const float xl = e.lF - e.lG * xnext - e.lH * xf;
        if (nvalid > M) chunk_finish_smem<M, true, CW>(dv, tq, xf, xl, smL + j0 * CW + cx, nvalid);
        else chunk_finish_smem<M, false, CW>(dv, tq, xf, xl, smL + j0 * CW + cx, nvalid);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < nbox; ++b) tma_store_3d(&tmU, x0, b * BR, img, smL + b * BR * CW);
        bulk_commit_and_wait_read();
    }
    (void)U;
    (void)u_stride;
}

// Persistent form of k_aos_cols_tma: one CTA per SM walks the launch's strips round-robin with TWO shared-memory
// (L, c) strip buffers and a separate U staging strip.  A strip's L and c are in registers once its chunk
// reductions are done, so right after that barrier the buffer is refilled with strip i + 2 — its tensor copies
// stream in during the rest of strip i and all of strip i + 1 (the per-strip CTA above waited for its copies with
// only one other CTA per SM to fill the gap: 34% of its stalls were that barrier wait).  U leaves from the staging
// strip with tensor stores; the next strip's finish writes it only after they have read it.  After the reductions
// the chunk equations go to shared memory once and a warp per column forms its reduced rows and solves them with
// warp_pcr64 (no CTA barriers inside the solve): three barriers per strip in all.  One CTA of 16 warps per SM (the
// two strip buffers take 154 KB); 4-column strips at two CTAs per SM measured slower (28.2 vs 24.7 ms), and so did
// the per-strip CTA (two per SM, single-buffered) with this warp PCR (27.7 vs 24.9: 64 registers spill).
constexpr int kEP = 68;  // warp-PCR row pitch (floats)

template <int CW, int M, int NT>
__global__ void __launch_bounds__(NT, 1) k_aos_cols_tmap(const __grid_constant__ CUtensorMap tmL,
                                                         const __grid_constant__ CUtensorMap tmC,
                                                         const __grid_constant__ CUtensorMap tmU, Geom g, float tau,
                                                         int T, int TP, int nbox, int BR, int nsx, int nimg,
                                                         int total) {
    KZ_PDL_PROLOGUE();
    extern __shared__ __align__(128) float smem_cols[];
    __shared__ __align__(8) uint64_t bar[2];
    const int HB = nbox * BR;
    float* smU = smem_cols + 4 * HB * CW;  // after [2][L, c][HB][CW]
    float* Q = smU + HB * CW;              // chunk equations [CW][A, C, D, lF, lG, lH][kEP]
    float* X = Q + CW * 6 * kEP;           // reduced-system solutions [CW][kEP]
    const int G = gridDim.x;
    auto issue = [&](int w, int b) {
        const int z = w / nsx, x0 = (w - z * nsx) * CW, img = batch_image(z, nimg, g);
        float* dL = smem_cols + 2 * b * HB * CW;
        float* dC = dL + HB * CW;
        mbar_arrive_expect_tx(&bar[b], 2u * (uint32_t)(HB * CW) * 4u);
        for (int q = 0; q < nbox; ++q) {
            tma_load_3d(dL + q * BR * CW, &tmL, x0, q * BR, img, &bar[b]);
            tma_load_3d(dC + q * BR * CW, &tmC, x0, q * BR, img, &bar[b]);
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        if ((int)blockIdx.x < total) issue(blockIdx.x, 0);
        if ((int)blockIdx.x + G < total) issue(blockIdx.x + G, 1);
    }
    __syncthreads();  // the barriers are initialised before anyone waits on them
    const int cx = threadIdx.x % CW, p = threadIdx.x / CW;
    const int n = g.H;
    const int j0 = p * M;
    const int nvalid = n - j0;
    int it = 0;
    for (int w = blockIdx.x; w < total; w += G, ++it) {
        const int b = it & 1;
        const int z = w / nsx, x0 = (w - z * nsx) * CW, img = batch_image(z, nimg, g);
        const float* smL = smem_cols + 2 * b * HB * CW;
        const float* smC = smL + HB * CW;
        const bool active = (p < T) && (x0 + cx < g.W);
        float dv[M], tq[M + 1];
        ChunkEq e{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        mbar_wait(&bar[b], (uint32_t)((it >> 1) & 1));
        if (active) {
            float cv[M];
            const bool full = nvalid > M;
            if (full) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    dv[i] = smL[(j0 + i) * CW + cx];
                    cv[i] = smC[(j0 + i) * CW + cx];
                }
            } else {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    dv[i] = i < nvalid ? smL[(j0 + i) * CW + cx] : 0.f;
                    cv[i] = i < nvalid ? smC[(j0 + i) * CW + cx] : 0.f;
                }
            }
            const float cprev = j0 > 0 ? smC[(j0 - 1) * CW + cx] : 0.f;
            tq[0] = j0 > 0 ? tau * (cprev + cv[0]) : 0.f;
            if (full) {
#pragma unroll
                for (int i = 1; i < M; ++i) tq[i] = tau * (cv[i - 1] + cv[i]);
                tq[M] = tau * (cv[M - 1] + smC[(j0 + M) * CW + cx]);
            } else {
#pragma unroll
                for (int i = 1; i < M; ++i) tq[i] = i < nvalid ? tau * (cv[i - 1] + cv[i]) : 0.f;
                tq[M] = 0.f;
            }
            chunk_reduce<M>(dv, tq, e);
        }
        // chunk equations → Q[cx][A, C, D, lF, lG, lH][p] (pitch kEP ≡ 4 mod 32: the 8 columns x 4 chunks of a warp
        // hit 32 distinct banks); a warp per column forms the reduced rows from them and solves them (warp PCR)
        {
            float* Qc = Q + cx * 6 * kEP;
            Qc[p] = e.A;
            Qc[kEP + p] = e.C;
            Qc[2 * kEP + p] = e.D;
            Qc[3 * kEP + p] = e.lF;
            Qc[4 * kEP + p] = e.lG;
            Qc[5 * kEP + p] = e.lH;
        }
        __syncthreads();  // every thread holds its strip samples in registers: refill the buffer with strip i + 2
        if (threadIdx.x == 0 && w + 2 * G < total) issue(w + 2 * G, b);
        {
            // warp wq solves columns wq, wq + nw, ... (CW·TP/32 warps; 16 at 64 chunks, so one column each); row r of
            // column q couples chunk r with chunk r − 1's last equation; rows of padding chunks / columns past the
            // image are identity rows (exactly as the per-strip kernel builds them)
            const int wq = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = (CW * TP) >> 5;
            for (int q = wq; q < CW; q += nw) {
                const float* Qq = Q + q * 6 * kEP;
                const bool col = x0 + q < g.W;
                float ra[2], rb[2], rc[2], rd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int r = 2 * ln + u;
                    ra[u] = 0.f;
                    rb[u] = 1.f;
                    rc[u] = 0.f;
                    rd[u] = 0.f;
                    if (col && r < T) {
                        const float A = Qq[r], C = Qq[kEP + r], D = Qq[2 * kEP + r];
                        const float lF = Qq[3 * kEP + r], lG = Qq[4 * kEP + r], lH = Qq[5 * kEP + r];
                        float pF = 0.f, pG = 0.f, pH = 0.f;
                        if (r > 0) {
                            pF = Qq[3 * kEP + r - 1];
                            pG = Qq[4 * kEP + r - 1];
                            pH = Qq[5 * kEP + r - 1];
                        }
                        ra[u] = -A * pH;
                        rb[u] = 1.f - A * pG - C * lH;
                        rc[u] = -C * lG;
                        rd[u] = D - A * pF - C * lF;
                    }
                }
                *reinterpret_cast<float2*>(X + q * kEP + 2 * ln) = warp_pcr64(ra, rb, rc, rd, ln);
            }
        }
        // the previous strip's U stores must have read the staging strip before this strip's finish rewrites it
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        const float xf = X[cx * kEP + p];
        if (active) {
            const float xnext = (p + 1 < T) ? X[cx * kEP + p + 1] : 0.f;
            const float xl = e.lF - e.lG * xnext - e.lH * xf;
            if (nvalid > M) chunk_finish_smem<M, true, CW>(dv, tq, xf, xl, smU + j0 * CW + cx, nvalid);
            else chunk_finish_smem<M, false, CW>(dv, tq, xf, xl, smU + j0 * CW + cx, nvalid);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < nbox; ++q) tma_store_3d(&tmU, x0, q * BR, img, smU + q * BR * CW);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// -------------------------------------------------------------------------------------------------------------
// Row systems, one CTA of NW warps per row (the row pass runs first and writes V).  The TMA engine streams the
// row's L and c into shared memory; thread p owns the chunk [p·M, p·M + m) (M odd: conflict-free strided reads)
// and eliminates it in registers; the reduced system (one unknown per thread) is solved by a warp-level SPIKE:
// shuffle PCR inside each warp on three right-hand sides, a serial 2·NW-unknown boundary solve by one thread,
// then x = y − v·x_{prev warp} − z·x_{next warp}.  x goes back to shared memory and V leaves with 16-byte stores.
template <int M, int NW>
__global__ void __launch_bounds__(32 * NW) k_aos_rows_cta(const float* __restrict__ L, const float* __restrict__ c,
                                                          const float* __restrict__ U, float* __restrict__ Lout,
                                                          Strides st, Geom g, float tau, int T) {
    KZ_PDL_PROLOGUE();
    constexpr int MC = M + 1, TP = 32 * NW;
    extern __shared__ __align__(16) float rs[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ float lastA[TP], lastG[TP], lastD[TP], bnd[NW * 6], sol[NW * 2], fx[TP];
    const int n = g.W;
    const int Wp = (n + 3) & ~3;
    float* sL = rs;
    float* sC = rs + Wp;
    float* sU = rs + 2 * Wp;
    const int p = threadIdx.x, lane = p & 31, w = p >> 5;
    const int q = g.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;  // descending: last image's last row first
    const int img = q / g.H, y = q - img * g.H;
    const size_t ry = (size_t)y * g.P;
    if (p == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 12u * (uint32_t)Wp);
        bulk_g2s(sL, L + img * st.L + ry, 4u * (uint32_t)Wp, &bar);
        bulk_g2s(sC, c + img * st.c + ry, 4u * (uint32_t)Wp, &bar);
        bulk_g2s(sU, U + img * st.U + ry, 4u * (uint32_t)Wp, &bar);
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
    // L_i = ½(U + V), U from the column pass
    float4* Or = reinterpret_cast<float4*>(Lout + img * st.out + ry);
    for (int v = p; v < (Wp >> 2); v += TP) {
        const float4 a = reinterpret_cast<const float4*>(sL)[v], b = reinterpret_cast<const float4*>(sU)[v];
        Or[v] = make_float4(0.5f * (a.x + b.x), 0.5f * (a.y + b.y), 0.5f * (a.z + b.z), 0.5f * (a.w + b.w));
    }
}

template <int M, int NW>
void run_rows_cta(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg, float tau,
                  cudaStream_t s) {
    int T = (g.W + M - 1) / M;
    if (T > 1 && g.W - (T - 1) * M == 1) --T;
    const size_t smem = sizeof(float) * 3 * ((g.W + 3) & ~3);
    ensure_smem_optin(reinterpret_cast<const void*>(k_aos_rows_cta<M, NW>), (int)smem);  // + static smem may pass 48 KB
    kz_launch(k_aos_rows_cta<M, NW>, dim3(g.H * nimg), dim3(32 * NW), smem, s, L, c, U, Lout, st, g, tau, T);
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// 3-D fp32 map over nimg planes of W x H (row pitch P floats, plane stride `plane_stride` floats), box CW x BR x 1.
bool encode_plane_map(CUtensorMap* m, const float* base, Geom g, int nimg, size_t plane_stride, int CW, int BR) {
    const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)nimg};
    const cuuint64_t strides[2] = {(cuuint64_t)g.P * 4, (cuuint64_t)plane_stride * 4};
    const cuuint32_t box[3] = {(cuuint32_t)CW, (cuuint32_t)BR, 1};
    return encode_f32_map(m, 3, base, dims, strides, box);
}

template <int CW, int M, int NT, int MINB>
bool run_cols_tma(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau, cudaStream_t s) {
    const int T = (g.H + M - 1) / M;
    const int TP = round_up(T, 32 / CW);
    if (CW * TP > NT) return false;
    // boxes of BR rows, BR a multiple of 4 (CW = 8 floats x 4 rows = 128 B: every box lands 128-byte aligned)
    const int nbox = (g.H + 255) / 256, BR = round_up((g.H + nbox - 1) / nbox, 4);
    CUtensorMap tmL, tmC, tmU;
    if (!encode_plane_map(&tmL, L, g, nimg, st.L, CW, BR) || !encode_plane_map(&tmC, c, g, nimg, st.c, CW, BR) ||
        !encode_plane_map(&tmU, U, g, nimg, st.out, CW, BR))
        return false;
    const size_t smem = sizeof(float) * (2 * (size_t)nbox * BR * CW + 7 * (size_t)CW * TP);
    if (!ensure_smem_optin(reinterpret_cast<const void*>(k_aos_cols_tma<CW, M, NT, MINB>), (int)smem)) return false;
    dim3 grid((g.W + CW - 1) / CW, 1, nimg);
    kz_launch(k_aos_cols_tma<CW, M, NT, MINB>, dim3(grid), dim3(CW * TP), smem, s, tmL, tmC, tmU, U, st.out, g, tau,
              T, TP, nbox, BR);
    return true;
}

template <int CW, int M, int NT>
bool run_cols_tmap(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau, cudaStream_t s) {
    const int T = (g.H + M - 1) / M;
    const int TP = round_up(T, 32 / CW);
    if (CW * TP > NT) return false;
    const int nbox = (g.H + 255) / 256, BR = round_up((g.H + nbox - 1) / nbox, 4);
    CUtensorMap tmL, tmC, tmU;
    if (!encode_plane_map(&tmL, L, g, nimg, st.L, CW, BR) || !encode_plane_map(&tmC, c, g, nimg, st.c, CW, BR) ||
        !encode_plane_map(&tmU, U, g, nimg, st.out, CW, BR))
        return false;
    if (TP > 64) return false;  // the warp PCR holds 64 chunk unknowns per column
    const size_t smem = sizeof(float) * (5 * (size_t)nbox * BR * CW + (size_t)CW * 7 * kEP);
    if (!ensure_smem_optin(reinterpret_cast<const void*>(k_aos_cols_tmap<CW, M, NT>), (int)smem)) return false;
    const int nsx = (g.W + CW - 1) / CW, total = nsx * nimg;
    const int grid = std::min(total, device_sm_count());
    kz_launch(k_aos_cols_tmap<CW, M, NT>, dim3(grid), dim3(CW * TP), smem, s, tmL, tmC, tmU, g, tau, T, TP, nbox, BR,
              nsx, nimg, total);
    return true;
}

template <int CW, int M, int NT, int MINB>
void run_cols(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau, cudaStream_t s) {
    const int T = (g.H + M - 1) / M;  // the last chunk is padded (decoupled rows)
    const int TP = round_up(T, 32 / CW);
    const size_t smem = sizeof(float) * 7 * CW * TP;
    ensure_smem_optin(reinterpret_cast<const void*>(k_aos_cols_u<CW, M, NT, MINB>), (int)smem);
    dim3 grid((g.W + CW - 1) / CW, 1, nimg);
    kz_launch(k_aos_cols_u<CW, M, NT, MINB>, dim3(grid), dim3(CW * TP), smem, s, L, c, U, st, g, tau, T, TP);
}

}  // namespace

// Column chunk length M: T = ceil(H/M) chunks per column, CW*TP <= NT threads; MINB = 2 keeps two CTAs resident
// per SM so one CTA's loads overlap the other's solve.  At 1920x1200 (256-image step, 1 B200): M = 20 (480
// threads, 64 registers) 34.7 ms, M = 24 (72 registers) 39.7 ms, M = 16 (608 threads, one CTA per SM) 45.8 ms.
bool launch_aos_cols(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau,
                     cudaStream_t s) {
    const int H = g.H;
    static const int tma = tune_knob("KAZE_COLS_TMA", 1);
    // TMA-staged inputs, odd chunk lengths (conflict-free shared reads), <= 64 chunks per column
    static const int persistent = tune_knob("KAZE_COLS_PERSIST", 1);
    if (tma && persistent && H <= 64 * 19) {
        bool ok;
        // (smaller chunks with more threads measured slower: M = 11 x 128 chunks 32.3 ms, M = 13 x 96 30.8, vs 27.1
        // at M = 19 x 64 — one more PCR level and its barriers; with the warp PCR, 4-column strips at two CTAs per SM
        // 28.2 vs 24.7 ms)
        if (H <= 64 * 9) ok = run_cols_tmap<8, 9, 512>(L, c, U, st, g, nimg, tau, s);
        else if (H <= 64 * 13) ok = run_cols_tmap<8, 13, 512>(L, c, U, st, g, nimg, tau, s);
        else if (H <= 64 * 17) ok = run_cols_tmap<8, 17, 512>(L, c, U, st, g, nimg, tau, s);
        else ok = run_cols_tmap<8, 19, 512>(L, c, U, st, g, nimg, tau, s);
        if (ok) return true;
    }
    if (tma && H <= 64 * 19) {
        bool ok;
        if (H <= 64 * 9) ok = run_cols_tma<8, 9, 512, 2>(L, c, U, st, g, nimg, tau, s);
        else if (H <= 64 * 13) ok = run_cols_tma<8, 13, 512, 2>(L, c, U, st, g, nimg, tau, s);
        else if (H <= 64 * 17) ok = run_cols_tma<8, 17, 512, 2>(L, c, U, st, g, nimg, tau, s);
        else ok = run_cols_tma<8, 19, 512, 2>(L, c, U, st, g, nimg, tau, s);
        if (ok) return true;
    }
    if (H <= 8 * 64) run_cols<8, 8, 512, 2>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 12 * 64) run_cols<8, 12, 512, 2>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 16 * 64) run_cols<8, 16, 512, 2>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 20 * 64) run_cols<8, 20, 512, 2>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 32 * 64) run_cols<4, 32, 256, 2>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 32 * 128) run_cols<4, 32, 512, 1>(L, c, U, st, g, nimg, tau, s);
    else if (H <= 32 * 256) run_cols<2, 32, 512, 1>(L, c, U, st, g, nimg, tau, s);
    else return false;
    return true;
}

// Row systems, one CTA per row: the smallest odd chunk M >= 5 with T = ceil(W/M) <= 32·NW threads.
bool launch_aos_rows(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg,
                     float tau, cudaStream_t s) {
    const int W = g.W;
    if (W <= 128 * 5) run_rows_cta<5, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 128 * 7) run_rows_cta<7, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 128 * 9) run_rows_cta<9, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 128 * 11) run_rows_cta<11, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 128 * 13) run_rows_cta<13, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 128 * 15) run_rows_cta<15, 4>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 11) run_rows_cta<11, 8>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 17) run_rows_cta<17, 8>(L, c, U, Lout, st, g, nimg, tau, s);
    else if (W <= 256 * 33) run_rows_cta<33, 8>(L, c, U, Lout, st, g, nimg, tau, s);
    else return false;
    return true;
}

}  // namespace kz
