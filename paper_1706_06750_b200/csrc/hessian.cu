// hessian.cu — multiscale derivatives and the scale-normalised Hessian determinant (Eq. 8; A9, A10).
//
// With the dilated Scharr operator at step s (taps at 0, ±s; derivative (−1, 0, 1)/2 after the s-normalisation,
// cross smoothing (3, 10, 3)/16) written N_x, N_y:
//     Lx = N_x L,  Ly = N_y L,  Ldet = N_x(Lx)·N_y(Ly) − N_y(Lx)²
// which equals s⁴(LxxLyy − Lxy²) with per-pixel derivatives (the factor s per derivative order is absorbed in
// N).  Second derivatives read the MATERIALISED first derivatives at clamped coordinates (A10), so they are two
// passes: hess_first (L → Lx, Ly) and hess_det (Lx, Ly → Ldet).  One launch covers every level of every image
// (blockIdx.y packs (level, row-tile)); the per-level step s_i comes from the LevelTable.
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr float kW0 = 0.1875f, kW1 = 0.625f;  // (3, 10, 3) / 16

// Two-pass form, one launch per pass for ALL levels (blockIdx.y packs (level, 32-row tile)).  A thread computes
// four outputs (rows ty, ty+8, ty+16, ty+24 of a 32x32 tile); the eight ring taps at distance s are fixed 32-bit
// offsets from the output address, so interior tiles issue plain loads with no clamping or 64-bit index math.
__global__ void __launch_bounds__(256) k_hess_first(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                    size_t img_stride, Geom g, LevelTable lt, int tiles_y) {
    const int level = blockIdx.y / tiles_y, ty_t = blockIdx.y - level * tiles_y;
    const int s = lt.step[level];
    const int x = blockIdx.x * 32 + threadIdx.x, yb = ty_t * 32 + threadIdx.y;
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float* L = Lt + base;
    float2* D = Lxy + base;
    const bool interior = (blockIdx.x * 32 >= s) && (blockIdx.x * 32 + 32 + s <= g.W) && (ty_t * 32 >= s) &&
                          (ty_t * 32 + 32 + s <= g.H);
    if (interior) {
        const int P = g.P, sp = s * P;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int y = yb + 8 * k;
            const float* q = L + (size_t)y * P + x;
            const float a = __ldg(q - sp - s), b = __ldg(q - sp), c = __ldg(q - sp + s);
            const float d = __ldg(q - s), f = __ldg(q + s);
            const float h = __ldg(q + sp - s), i = __ldg(q + sp), j = __ldg(q + sp + s);
            D[(size_t)y * P + x] = make_float2(0.5f * (kW0 * (c - a) + kW1 * (f - d) + kW0 * (j - h)),
                                               0.5f * (kW0 * (h - a) + kW1 * (i - b) + kW0 * (j - c)));
        }
        return;
    }
    if (x >= g.W) return;
    const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int y = yb + 8 * k;
        if (y >= g.H) break;
        const int ym = max(y - s, 0), yp = min(y + s, g.H - 1);
        const float* rm = L + (size_t)ym * g.P;
        const float* r0 = L + (size_t)y * g.P;
        const float* rp = L + (size_t)yp * g.P;
        const float a = __ldg(rm + xm), b = __ldg(rm + x), c = __ldg(rm + xp);
        const float d = __ldg(r0 + xm), f = __ldg(r0 + xp);
        const float h = __ldg(rp + xm), i = __ldg(rp + x), j = __ldg(rp + xp);
        D[(size_t)y * g.P + x] = make_float2(0.5f * (kW0 * (c - a) + kW1 * (f - d) + kW0 * (j - h)),
                                             0.5f * (kW0 * (h - a) + kW1 * (i - b) + kW0 * (j - c)));
    }
}

__device__ __forceinline__ float det_from_ring(float2 a, float2 b, float2 c, float2 d, float2 f, float2 h, float2 i,
                                               float2 j) {
    const float lxx = 0.5f * (kW0 * (c.x - a.x) + kW1 * (f.x - d.x) + kW0 * (j.x - h.x));  // N_x(Lx)
    const float lxy = 0.5f * (kW0 * (h.x - a.x) + kW1 * (i.x - b.x) + kW0 * (j.x - c.x));  // N_y(Lx)
    const float lyy = 0.5f * (kW0 * (h.y - a.y) + kW1 * (i.y - b.y) + kW0 * (j.y - c.y));  // N_y(Ly)
    return lxx * lyy - lxy * lxy;
}

__global__ void __launch_bounds__(256) k_hess_det(const float2* __restrict__ Lxy, float* __restrict__ Ldet,
                                                  size_t img_stride, Geom g, LevelTable lt, int tiles_y) {
    const int level = blockIdx.y / tiles_y, ty_t = blockIdx.y - level * tiles_y;
    const int s = lt.step[level];
    const int x = blockIdx.x * 32 + threadIdx.x, yb = ty_t * 32 + threadIdx.y;
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float2* D = Lxy + base;
    float* O = Ldet + base;
    const bool interior = (blockIdx.x * 32 >= s) && (blockIdx.x * 32 + 32 + s <= g.W) && (ty_t * 32 >= s) &&
                          (ty_t * 32 + 32 + s <= g.H);
    if (interior) {
        const int P = g.P, sp = s * P;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int y = yb + 8 * k;
            const float2* q = D + (size_t)y * P + x;
            O[(size_t)y * P + x] = det_from_ring(__ldg(q - sp - s), __ldg(q - sp), __ldg(q - sp + s), __ldg(q - s),
                                                 __ldg(q + s), __ldg(q + sp - s), __ldg(q + sp), __ldg(q + sp + s));
        }
        return;
    }
    if (x >= g.W) return;
    const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int y = yb + 8 * k;
        if (y >= g.H) break;
        const int ym = max(y - s, 0), yp = min(y + s, g.H - 1);
        const size_t om = (size_t)ym * g.P, o0 = (size_t)y * g.P, op = (size_t)yp * g.P;
        O[o0 + x] = det_from_ring(__ldg(D + om + xm), __ldg(D + om + x), __ldg(D + om + xp), __ldg(D + o0 + xm),
                                  __ldg(D + o0 + xp), __ldg(D + op + xm), __ldg(D + op + x), __ldg(D + op + xp));
    }
}

// Fused per-level Hessian: one CTA computes a T x T output tile of Lx, Ly and Ldet, with the L tile (T + 4S)² and
// the first-derivative tile (T + 2S)² in shared memory — 16 B/px of DRAM traffic instead of 24 B/px for the
// two-pass form.  The step S is a template parameter (one instantiation per step of the schedule), so every index
// is compile-time affine.  Virtual coordinates outside the image are evaluated at their clamped position, which is
// exactly what the clamped-intermediate semantics (A10) read; interior tiles skip all clamping.
template <int T, int S>
__global__ void __launch_bounds__(T * 8) k_hess_fused(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                      float* __restrict__ Ldet, size_t img_stride, Geom g) {
    constexpr int NL = T + 4 * S, ND = T + 2 * S;
    constexpr int NLP = NL | 1;  // odd pitches: column walks by a warp are conflict free
    extern __shared__ __align__(16) float hsm[];
    float* tL = hsm;                                                   // NL x NLP
    float2* tD = reinterpret_cast<float2*>(hsm + ((NL * NLP + 3) & ~3));  // ND x ND
    const int x0 = blockIdx.x * T, y0 = blockIdx.y * T;
    const size_t base = blockIdx.z * img_stride;
    const float* L = Lt + base;
    const int tx = threadIdx.x, ty = threadIdx.y;  // blockDim = (T, 8)
    const bool interior = (x0 - 2 * S >= 0) && (y0 - 2 * S >= 0) && (x0 + T + 2 * S <= g.W) && (y0 + T + 2 * S <= g.H);
    // ---- L tile ----
    constexpr int KC = (NL + T - 1) / T;
    for (int r = ty; r < NL; r += 8) {
        const float* row = L + (size_t)(interior ? y0 - 2 * S + r : clampi(y0 - 2 * S + r, 0, g.H - 1)) * g.P;
        float v[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int cidx = tx + k * T;
            const int gx = interior ? x0 - 2 * S + cidx : clampi(x0 - 2 * S + cidx, 0, g.W - 1);
            v[k] = (cidx < NL) ? __ldg(row + gx) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < KC; ++k)
            if (tx + k * T < NL) tL[r * NLP + tx + k * T] = v[k];
    }
    __syncthreads();
    // ---- first derivatives on the ND x ND tile (virtual coords y0-S.., x0-S..) ----
    constexpr int KD = (ND + T - 1) / T;
    for (int r = ty; r < ND; r += 8) {
        int ym, y1, yp;
        if (interior) {
            y1 = r + S;
            ym = r;
            yp = r + 2 * S;
        } else {
            const int vy = clampi(y0 - S + r, 0, g.H - 1);
            y1 = vy - (y0 - 2 * S);
            ym = clampi(vy - S, 0, g.H - 1) - (y0 - 2 * S);
            yp = clampi(vy + S, 0, g.H - 1) - (y0 - 2 * S);
        }
#pragma unroll
        for (int k = 0; k < KD; ++k) {
            const int cidx = tx + k * T;
            if (cidx >= ND) continue;
            int xm, x1, xp;
            if (interior) {
                x1 = cidx + S;
                xm = cidx;
                xp = cidx + 2 * S;
            } else {
                const int vx = clampi(x0 - S + cidx, 0, g.W - 1);
                x1 = vx - (x0 - 2 * S);
                xm = clampi(vx - S, 0, g.W - 1) - (x0 - 2 * S);
                xp = clampi(vx + S, 0, g.W - 1) - (x0 - 2 * S);
            }
            const float a = tL[ym * NLP + xm], b = tL[ym * NLP + x1], c = tL[ym * NLP + xp];
            const float d = tL[y1 * NLP + xm], f = tL[y1 * NLP + xp];
            const float h = tL[yp * NLP + xm], ii = tL[yp * NLP + x1], j = tL[yp * NLP + xp];
            const float dx = 0.5f * (kW0 * (c - a) + kW1 * (f - d) + kW0 * (j - h));
            const float dy = 0.5f * (kW0 * (h - a) + kW1 * (ii - b) + kW0 * (j - c));
            tD[r * ND + cidx] = make_float2(dx, dy);
        }
    }
    __syncthreads();
    // ---- outputs: Lx, Ly (centre of tD) and Ldet ----
    const int x = x0 + tx;
    int xm = tx, x1 = tx + S, xp = tx + 2 * S;
    if (!interior) {
        xm = clampi(x - S, 0, g.W - 1) - (x0 - S);
        xp = clampi(x + S, 0, g.W - 1) - (x0 - S);
    }
    float2* Dout = Lxy + base;
    float* Lout = Ldet + base;
#pragma unroll 4
    for (int r = ty; r < T; r += 8) {
        const int y = y0 + r;
        int ym = r, y1 = r + S, yp = r + 2 * S;
        if (!interior) {
            ym = clampi(y - S, 0, g.H - 1) - (y0 - S);
            yp = clampi(y + S, 0, g.H - 1) - (y0 - S);
        }
        const float2 a = tD[ym * ND + xm], b = tD[ym * ND + x1], c = tD[ym * ND + xp];
        const float2 d = tD[y1 * ND + xm], e = tD[y1 * ND + x1], f = tD[y1 * ND + xp];
        const float2 h = tD[yp * ND + xm], ii = tD[yp * ND + x1], j = tD[yp * ND + xp];
        const float lxx = 0.5f * (kW0 * (c.x - a.x) + kW1 * (f.x - d.x) + kW0 * (j.x - h.x));
        const float lxy = 0.5f * (kW0 * (h.x - a.x) + kW1 * (ii.x - b.x) + kW0 * (j.x - c.x));
        const float lyy = 0.5f * (kW0 * (h.y - a.y) + kW1 * (ii.y - b.y) + kW0 * (j.y - c.y));
        if (x < g.W && y < g.H) {
            Dout[(size_t)y * g.P + x] = e;
            Lout[(size_t)y * g.P + x] = lxx * lyy - lxy * lxy;
        }
    }
}

template <int T, int S>
void run_hess(const float* Lt, float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, cudaStream_t st) {
    constexpr int NL = T + 4 * S, ND = T + 2 * S, NLP = NL | 1;
    const size_t smem = sizeof(float) * (((NL * NLP + 3) & ~3) + 2 * ND * ND);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_hess_fused<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid((g.W + T - 1) / T, (g.H + T - 1) / T, nimg);
    k_hess_fused<T, S><<<grid, dim3(T, 8), smem, st>>>(Lt, Lxy, Ldet, img_stride, g);
}

__global__ void k_component_copy(float2* __restrict__ plane, int comp, float* __restrict__ tight, int to_tight,
                                 Geom g) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= g.W) return;
    float* e = reinterpret_cast<float*>(plane + (size_t)y * g.P + x) + comp;
    if (to_tight) tight[(size_t)y * g.W + x] = *e;
    else *e = tight[(size_t)y * g.W + x];
}

}  // namespace

void launch_hess_first(const float* Lt, float2* Lxy, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                       cudaStream_t s) {
    int ty = (g.H + 31) / 32;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_first<<<grid, dim3(32, 8), 0, s>>>(Lt, Lxy, img_stride, g, lt, ty);
}

void launch_hess_det(const float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                     cudaStream_t s) {
    int ty = (g.H + 31) / 32;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_det<<<grid, dim3(32, 8), 0, s>>>(Lxy, Ldet, img_stride, g, lt, ty);
}

bool launch_hessian(const float* Lt, float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, int step,
                    cudaStream_t st) {
    switch (step) {
#define KZ_H(S)                                                            \
    case S:                                                                \
        if (S <= 8) run_hess<32, S>(Lt, Lxy, Ldet, img_stride, g, nimg, st); \
        else run_hess<64, S>(Lt, Lxy, Ldet, img_stride, g, nimg, st);      \
        return true;
        KZ_H(1) KZ_H(2) KZ_H(3) KZ_H(4) KZ_H(5) KZ_H(6) KZ_H(7) KZ_H(8) KZ_H(9) KZ_H(10) KZ_H(11) KZ_H(12) KZ_H(13)
        KZ_H(14) KZ_H(15) KZ_H(16) KZ_H(17) KZ_H(18) KZ_H(19) KZ_H(20) KZ_H(21) KZ_H(22) KZ_H(23) KZ_H(24)
#undef KZ_H
        default: return false;
    }
}

void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s) {
    k_component_copy<<<dim3((g.W + 255) / 256, g.H), 256, 0, s>>>(plane, comp, tight, to_tight, g);
}

}  // namespace kz
