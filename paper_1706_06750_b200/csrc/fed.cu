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
