// fed.cu — FED scale-space backend: the explicit cycles of Eq. 5 (readings
// A20, A21) on sm_100a, selectable instead of the AOS step of Eq. 4 (kaze_params.scheme = KAZE_SCHEME_FED).
//
// One explicit step with the conductivities held fixed (A20):
//   L⁺_p = L_p + τ_j Σ_{q ∈ N4(p)} ½(c_p + c_q)(L_q − L_p),   faces on the image border carry no flux (Neumann).
// A cycle of n steps (τ_j of Eq. 5, scaled to reach t_i exactly, in the A21 κ order) takes L_{i−1} to L_i.
//
// Temporal blocking: one launch advances a 64x32 output tile by K <= 8 steps.  The CTA loads L and c over the tile
// plus a K-pixel halo (clamped reads keep the halo finite), turns c into per-face weights once (zero across the
// image border and outside it, so halo cells never leak into image cells), then runs the K steps in shared memory,
// each shrinking the valid region by one pixel, and writes only the tile.  HBM traffic per launch is one read of
// L and c and one write of L (12 B/px) for K steps instead of 12 B/px per step.
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr int FTW = 64, FTH = 32;  // output tile (64 x 64 measured 255 vs 252 ms per 256-image step)

template <int K>
__global__ void __launch_bounds__(256) k_fed(const float* __restrict__ Lin, size_t s_in, const float* __restrict__ c,
                                             size_t s_c, float* __restrict__ Lout, size_t s_out, Geom g,
                                             FedTaus taus) {
    KZ_PDL_PROLOGUE();
    constexpr int EW = FTW + 2 * K, EH = FTH + 2 * K, SP = EW + 1;
    extern __shared__ float sm[];
    float* A = sm;
    float* B = A + EH * SP;
    float* WX = B + EH * SP;  // face (x, x+1) of cell (ly, lx)
    float* WY = WX + EH * SP; // face (y, y+1)
    const int x0 = blockIdx.x * FTW - K, y0 = blockIdx.y * FTH - K, img = blockIdx.z;
    const float* Li = Lin + img * s_in;
    const float* ci = c + img * s_c;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    {   // all tile loads issued before any shared store (one load-then-store per iteration left the load phase
        // latency-bound: 31% of the stall samples on its first shared store)
        constexpr int NV = (EH * EW + 255) / 256;
        float va[NV], vb[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int i = tid + 256 * k;
            if (i < EH * EW) {
                const int ly = i / EW, lx = i - ly * EW;
                const size_t gi = (size_t)clampi(y0 + ly, 0, g.H - 1) * g.P + clampi(x0 + lx, 0, g.W - 1);
                va[k] = __ldg(Li + gi);
                vb[k] = __ldg(ci + gi);
            }
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int i = tid + 256 * k;
            if (i < EH * EW) {
                const int ly = i / EW, lx = i - ly * EW;
                A[ly * SP + lx] = va[k];
                B[ly * SP + lx] = vb[k];
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < EH * EW; i += 256) {
        const int ly = i / EW, lx = i - ly * EW;
        const int gx = x0 + lx, gy = y0 + ly;
        const bool in = gx >= 0 && gx < g.W && gy >= 0 && gy < g.H;
        const float cp = B[ly * SP + lx];
        WX[ly * SP + lx] = (in && lx + 1 < EW && gx + 1 < g.W) ? 0.5f * (cp + B[ly * SP + lx + 1]) : 0.f;
        WY[ly * SP + lx] = (in && ly + 1 < EH && gy + 1 < g.H) ? 0.5f * (cp + B[(ly + 1) * SP + lx]) : 0.f;
    }
    __syncthreads();
    float* src = A;
    float* dst = B;
#pragma unroll 1
    for (int s = 1; s <= K; ++s) {
        const float tau = taus.t[s - 1];
        // thread (tx, ty): columns s + tx + 32k, and a contiguous eighth of the rows [s, EH - s), walked downwards
        // with the cell above and its face weight kept in registers (6 shared loads per cell instead of 9).
        // (Column pairs in fp32x2 from 8-byte shared loads — 6 loads per two cells — measured 264.6 vs 252 ms.)
        const int nrow = EH - 2 * s, per = (nrow + 7) / 8;
        const int r0 = s + ty * per, r1 = min(r0 + per, EH - s);
        for (int lx = s + tx; lx < EW - s; lx += 32) {
            if (r0 >= r1) break;
            int o = r0 * SP + lx;
            float up = src[o - SP], wyu = WY[o - SP], v = src[o];
            for (int ly = r0; ly < r1; ++ly, o += SP) {
                const float dn = src[o + SP], wy = WY[o];
                const float f = WX[o] * (src[o + 1] - v) - WX[o - 1] * (v - src[o - 1]) + wy * (dn - v) -
                                wyu * (v - up);
                dst[o] = fmaf(tau, f, v);
                up = v;
                v = dn;
                wyu = wy;
            }
        }
        __syncthreads();
        float* t = src;
        src = dst;
        dst = t;
    }
    float* Lo = Lout + img * s_out;
    for (int ly = K + ty; ly < K + FTH; ly += 8) {
        const int gy = y0 + ly;
        if (gy >= g.H) break;
        for (int lx = K + tx; lx < K + FTW; lx += 32) {
            const int gx = x0 + lx;
            if (gx < g.W) Lo[(size_t)gy * g.P + gx] = src[ly * SP + lx];
        }
    }
}

// Register-blocked form (default): the CTA's region is 64 columns x 8R rows; lane l of warp w holds the column pair
// (2l, 2l+1) of rows wR .. wR+R−1 and their face weights in REGISTERS for all K steps.  Per step a row's horizontal
// neighbours come from the adjacent lanes (two shuffles per row and pair), its vertical ones from the thread's own
// rows except at the warp's first and last row, which are exchanged through shared memory (2 + 2 eight-byte
// accesses and one barrier per thread and step); the shared-memory kernel above spent 6 loads and a store per
// cell and step.  Outside the image and across its border the face weights are 0 (Neumann; halo cells stay
// finite and never leak in), the region edges likewise; after K steps the inner (64 − 2KH) x (8R − 2KH) cells are
// exact and written (halo KH = K rounded up to even: column pairs stay 8-byte aligned).
constexpr int kFedR = 8;  // rows per thread

template <int K>
__global__ void __launch_bounds__(256, 3) k_fed_reg(const float* __restrict__ Lin, size_t s_in,
                                                    const float* __restrict__ c, size_t s_c, float* __restrict__ Lout,
                                                    size_t s_out, Geom g, FedTaus taus) {
    KZ_PDL_PROLOGUE();
    // halo KH >= K, even, so every column pair starts 8-byte aligned (the region starts at an even column)
    constexpr int R = kFedR, KH = (K + 1) & ~1, TOW = 64 - 2 * KH, TOH = 8 * R - 2 * KH;
    __shared__ float2 xch[2][2][8][32];  // [parity][first/last row][warp][lane]
    __shared__ float2 wyx[8][32];        // face weights below each warp's last row (set-up exchange)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int img = blockIdx.z;
    const int cx = blockIdx.x * TOW - KH + 2 * lane;        // column of a (b = cx + 1)
    const int ry0 = blockIdx.y * TOH - KH + warp * R;         // first row of this thread
    const float* Li = Lin + img * s_in;
    const float* ci = c + img * s_c;
    const bool pair_in = cx >= 0 && cx + 1 < g.W;           // both columns inside the image
    const int xa = clampi(cx, 0, g.W - 1), xb = clampi(cx + 1, 0, g.W - 1);
    float2 L[R], C[R];  // (a, b) pairs
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const size_t ro = (size_t)clampi(ry0 + r, 0, g.H - 1) * g.P;
        if (pair_in) {
            L[r] = __ldg(reinterpret_cast<const float2*>(Li + ro + cx));
            C[r] = __ldg(reinterpret_cast<const float2*>(ci + ro + cx));
        } else {
            L[r] = make_float2(__ldg(Li + ro + xa), __ldg(Li + ro + xb));
            C[r] = make_float2(__ldg(ci + ro + xa), __ldg(ci + ro + xb));
        }
    }
    // face weights: WXa (a|b), WXb (b|right); WY = (a, b) faces (row r | row r+1); zero across the image border,
    // outside it and at the region's edges
    const bool ina = cx >= 0 && cx < g.W, inb = cx + 1 >= 0 && cx + 1 < g.W, inr = cx + 2 >= 0 && cx + 2 < g.W;
    float2 WX[R];  // (a|b), (b|right)
    float2 WY[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int y = ry0 + r;
        const bool rin = y >= 0 && y < g.H;
        const float cr = __shfl_down_sync(0xffffffffu, C[r].x, 1);  // c of the right neighbour column
        // lane 31's (b|right) face is the region edge: 0, which also makes it the zero left flux of lane 0 below
        WX[r] = make_float2((rin && ina && inb) ? 0.5f * (C[r].x + C[r].y) : 0.f,
                            (rin && inb && inr && lane < 31) ? 0.5f * (C[r].y + cr) : 0.f);
        if (r + 1 < R) {
            const bool din = y + 1 >= 0 && y + 1 < g.H;
            WY[r] = make_float2((rin && din && ina) ? 0.5f * (C[r].x + C[r + 1].x) : 0.f,
                                (rin && din && inb) ? 0.5f * (C[r].y + C[r + 1].y) : 0.f);
        }
    }
    // the last row's downward faces need the next warp's first-row c; the first row's upward faces the previous
    // warp's last-row weights
    xch[0][0][warp][lane] = C[0];
    __syncthreads();
    {
        const int y = ry0 + R - 1;
        const bool rin = y >= 0 && y < g.H, din = y + 1 >= 0 && y + 1 < g.H && warp < 7;
        const float2 cn = warp < 7 ? xch[0][0][warp + 1][lane] : make_float2(0.f, 0.f);
        WY[R - 1] = make_float2((rin && din && ina) ? 0.5f * (C[R - 1].x + cn.x) : 0.f,
                                (rin && din && inb) ? 0.5f * (C[R - 1].y + cn.y) : 0.f);
        wyx[warp][lane] = WY[R - 1];
    }
    __syncthreads();
    const float2 wtop = warp > 0 ? wyx[warp - 1][lane] : make_float2(0.f, 0.f);  // faces above row 0
    // Flux form of the step: every face flux w·(L_q − L_p) is computed once and added to one cell, subtracted from
    // the other (the (a, b) pair in fp32x2: FADD2/FMUL2/FFMA2).  Horizontal: (a|b) in the lane, (b|right) with the
    // right lane's a, and the left face's flux is the left lane's (b|right) flux; vertical: the flux below row r is
    // carried to row r + 1 as its flux above.
#pragma unroll
    for (int s = 0; s < K; ++s) {  // unrolled: τ and the buffer parity are compile-time per step
        const float2 tau = make_float2(taus.t[s], taus.t[s]);
        const int par = s & 1;
        xch[par][0][warp][lane] = L[0];
        xch[par][1][warp][lane] = L[R - 1];
        __syncthreads();  // (the parity double buffer makes one barrier per step enough)
        const float2 up = warp > 0 ? xch[par][1][warp - 1][lane] : L[0];
        const float2 dn = warp < 7 ? xch[par][0][warp + 1][lane] : L[R - 1];
        float2 Fu = __fmul2_rn(wtop, __fadd2_rn(L[0], make_float2(-up.x, -up.y)));  // flux above row 0 (into it)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float2 v = L[r];
            const float right = __shfl_down_sync(0xffffffffu, v.x, 1);
            const float2 Fh = __fmul2_rn(WX[r], __fadd2_rn(make_float2(v.y, right), make_float2(-v.x, -v.y)));
            // (left|a) = the left lane's (b|right); lane 0 reads lane 31's, which is 0
            const float fl = __shfl_sync(0xffffffffu, Fh.y, (lane + 31) & 31);
            const float2 d = r + 1 < R ? L[r + 1] : dn;
            const float2 Fd = __fmul2_rn(WY[r], __fadd2_rn(d, make_float2(-v.x, -v.y)));  // flux below row r
            // div = (a|b) − (left|a) + below − above  for a;  (b|right) − (a|b) + below − above  for b
            const float2 div = __fadd2_rn(__fadd2_rn(Fh, make_float2(-fl, -Fh.x)), __fadd2_rn(Fd, make_float2(-Fu.x, -Fu.y)));
            L[r] = __ffma2_rn(tau, div, v);
            Fu = Fd;
        }
    }
    // write the exact inner region
    float* Lo = Lout + img * s_out;
    const bool wa = 2 * lane >= KH && 2 * lane < 64 - KH && cx < g.W;
    const bool wb = 2 * lane + 1 >= KH && 2 * lane + 1 < 64 - KH && cx + 1 < g.W;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int lr = warp * R + r, y = ry0 + r;
        if (lr < KH || lr >= 8 * R - KH || y >= g.H || y < 0) continue;
        float* o = Lo + (size_t)y * g.P + cx;
        if (wa && wb) *reinterpret_cast<float2*>(o) = L[r];
        else if (wa) o[0] = L[r].x;
        else if (wb) o[1] = L[r].y;
    }
}

template <int K>
void run_fed_reg(const float* Lin, size_t s_in, const float* c, size_t s_c, float* Lout, size_t s_out, Geom g,
                 int nimg, const FedTaus& t, cudaStream_t s) {
    constexpr int KH = (K + 1) & ~1, TOW = 64 - 2 * KH, TOH = 8 * kFedR - 2 * KH;
    dim3 grid((g.W + TOW - 1) / TOW, (g.H + TOH - 1) / TOH, nimg);
    kz_launch(k_fed_reg<K>, dim3(grid), dim3(256), 0, s, Lin, s_in, c, s_c, Lout, s_out, g, t);
}

template <int K>
void run_fed(const float* Lin, size_t s_in, const float* c, size_t s_c, float* Lout, size_t s_out, Geom g, int nimg,
             const FedTaus& t, cudaStream_t s) {
    constexpr int EW = FTW + 2 * K, EH = FTH + 2 * K, SP = EW + 1;
    const size_t smem = sizeof(float) * 4 * EH * SP;
    ensure_smem_optin(reinterpret_cast<const void*>(k_fed<K>), (int)smem);
    dim3 grid((g.W + FTW - 1) / FTW, (g.H + FTH - 1) / FTH, nimg);
    kz_launch(k_fed<K>, dim3(grid), dim3(dim3(32, 8)), smem, s, Lin, s_in, c, s_c, Lout, s_out, g, t);
}

}  // namespace

bool launch_fed_steps(const float* Lin, size_t s_in, const float* c, size_t s_c, float* Lout, size_t s_out, Geom g,
                      int nimg, const FedTaus& t, int nsteps, cudaStream_t s) {
    static const int reg = tune_knob("KAZE_FED_REG", 1);
    if (reg) {
        switch (nsteps) {
            case 1: run_fed_reg<1>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 2: run_fed_reg<2>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 3: run_fed_reg<3>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 4: run_fed_reg<4>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 5: run_fed_reg<5>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 6: run_fed_reg<6>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 7: run_fed_reg<7>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            case 8: run_fed_reg<8>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); return true;
            default: return false;
        }
    }
    switch (nsteps) {
        case 1: run_fed<1>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 2: run_fed<2>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 3: run_fed<3>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 4: run_fed<4>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 5: run_fed<5>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 6: run_fed<6>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 7: run_fed<7>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        case 8: run_fed<8>(Lin, s_in, c, s_c, Lout, s_out, g, nimg, t, s); break;
        default: return false;
    }
    return true;
}

}  // namespace kz
