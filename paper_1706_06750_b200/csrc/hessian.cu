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

__global__ void __launch_bounds__(256) k_hess_first(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                    size_t img_stride, Geom g, LevelTable lt, int tiles_y) {
    const int level = blockIdx.y / tiles_y, ty = blockIdx.y - level * tiles_y;
    const int x = blockIdx.x * 32 + threadIdx.x, y = ty * 8 + threadIdx.y;
    if (x >= g.W || y >= g.H) return;
    const int s = lt.step[level];
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float* L = Lt + base;
    const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
    const int ym = max(y - s, 0), yp = min(y + s, g.H - 1);
    const float* rm = L + (size_t)ym * g.P;
    const float* r0 = L + (size_t)y * g.P;
    const float* rp = L + (size_t)yp * g.P;
    float a = __ldg(rm + xm), b = __ldg(rm + x), c = __ldg(rm + xp);
    float d = __ldg(r0 + xm), f = __ldg(r0 + xp);
    float h = __ldg(rp + xm), i = __ldg(rp + x), j = __ldg(rp + xp);
    float dx = 0.5f * (kW0 * (c - a) + kW1 * (f - d) + kW0 * (j - h));
    float dy = 0.5f * (kW0 * (h - a) + kW1 * (i - b) + kW0 * (j - c));
    Lxy[base + (size_t)y * g.P + x] = make_float2(dx, dy);
}

__global__ void __launch_bounds__(256) k_hess_det(const float2* __restrict__ Lxy, float* __restrict__ Ldet,
                                                  size_t img_stride, Geom g, LevelTable lt, int tiles_y) {
    const int level = blockIdx.y / tiles_y, ty = blockIdx.y - level * tiles_y;
    const int x = blockIdx.x * 32 + threadIdx.x, y = ty * 8 + threadIdx.y;
    if (x >= g.W || y >= g.H) return;
    const int s = lt.step[level];
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float2* D = Lxy + base;
    const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
    const int ym = max(y - s, 0), yp = min(y + s, g.H - 1);
    const size_t om = (size_t)ym * g.P, o0 = (size_t)y * g.P, op = (size_t)yp * g.P;
    // the 8 ring taps at distance s (clamped), each an (Lx, Ly) pair
    const float2 a = __ldg(D + om + xm), b = __ldg(D + om + x), c = __ldg(D + om + xp);
    const float2 d = __ldg(D + o0 + xm), f = __ldg(D + o0 + xp);
    const float2 h = __ldg(D + op + xm), i = __ldg(D + op + x), j = __ldg(D + op + xp);
    const float lxx = 0.5f * (kW0 * (c.x - a.x) + kW1 * (f.x - d.x) + kW0 * (j.x - h.x));  // N_x(Lx)
    const float lxy = 0.5f * (kW0 * (h.x - a.x) + kW1 * (i.x - b.x) + kW0 * (j.x - c.x));  // N_y(Lx)
    const float lyy = 0.5f * (kW0 * (h.y - a.y) + kW1 * (i.y - b.y) + kW0 * (j.y - c.y));  // N_y(Ly)
    Ldet[base + o0 + x] = lxx * lyy - lxy * lxy;
}

// Fused per-level Hessian: one CTA computes a T x T output tile of Lx, Ly (written) and Ldet (written) with the
// L tile (T + 4s)² and the first-derivative tile (T + 2s)² in shared memory — 16 B/px of DRAM traffic instead of
// 24 B/px for the two-pass form.  Virtual coordinates outside the image are evaluated at their clamped position,
// which is exactly what the clamped-intermediate semantics (A10) read.
template <int T>
__global__ void __launch_bounds__(T == 32 ? 256 : 1024) k_hess_fused(const float* __restrict__ Lt,
                                                                     float2* __restrict__ Lxy,
                                                                     float* __restrict__ Ldet, size_t img_stride,
                                                                     Geom g, int level, int s) {
    extern __shared__ __align__(16) float hsm[];
    const int NL = T + 4 * s, ND = T + 2 * s;
    float* tL = hsm;                                         // NL x NL
    float2* tD = reinterpret_cast<float2*>(hsm + ((NL * NL + 3) & ~3));  // ND x ND
    const int x0 = blockIdx.x * T, y0 = blockIdx.y * T;
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float* L = Lt + base;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int total = NL * NL;
    for (int i0 = tid; i0 < total; i0 += 4 * nt) {  // four independent loads in flight per thread
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * nt;
            if (i < total) {
                const int r = i / NL, cidx = i - r * NL;
                v[k] = __ldg(L + (size_t)clampi(y0 - 2 * s + r, 0, g.H - 1) * g.P + clampi(x0 - 2 * s + cidx, 0, g.W - 1));
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * nt;
            if (i < total) tL[i] = v[k];
        }
    }
    __syncthreads();
    // first derivatives at the clamped position of every virtual coordinate of the ND x ND tile
    for (int i = tid; i < ND * ND; i += nt) {
        const int r = i / ND, cidx = i - r * ND;
        const int vy = clampi(y0 - s + r, 0, g.H - 1), vx = clampi(x0 - s + cidx, 0, g.W - 1);
        // L tile index of the clamped taps clamp(v ± s)
        const int ym = clampi(vy - s, 0, g.H - 1) - (y0 - 2 * s), y1 = vy - (y0 - 2 * s),
                  yp = clampi(vy + s, 0, g.H - 1) - (y0 - 2 * s);
        const int xm = clampi(vx - s, 0, g.W - 1) - (x0 - 2 * s), x1 = vx - (x0 - 2 * s),
                  xp = clampi(vx + s, 0, g.W - 1) - (x0 - 2 * s);
        const float a = tL[ym * NL + xm], b = tL[ym * NL + x1], c = tL[ym * NL + xp];
        const float d = tL[y1 * NL + xm], f = tL[y1 * NL + xp];
        const float h = tL[yp * NL + xm], ii = tL[yp * NL + x1], j = tL[yp * NL + xp];
        const float dx = 0.5f * (kW0 * (c - a) + kW1 * (f - d) + kW0 * (j - h));
        const float dy = 0.5f * (kW0 * (h - a) + kW1 * (ii - b) + kW0 * (j - c));
        tD[i] = make_float2(dx, dy);
    }
    __syncthreads();
    float2* Dout = Lxy + base;
    float* Lout = Ldet + base;
    for (int i = tid; i < T * T; i += nt) {
        const int r = i / T, cidx = i - r * T;
        const int y = y0 + r, x = x0 + cidx;
        if (x >= g.W || y >= g.H) continue;
        const int ym = clampi(y - s, 0, g.H - 1) - (y0 - s), y1 = y - (y0 - s), yp = clampi(y + s, 0, g.H - 1) - (y0 - s);
        const int xm = clampi(x - s, 0, g.W - 1) - (x0 - s), x1 = x - (x0 - s), xp = clampi(x + s, 0, g.W - 1) - (x0 - s);
        const float2 a = tD[ym * ND + xm], b = tD[ym * ND + x1], c = tD[ym * ND + xp];
        const float2 d = tD[y1 * ND + xm], e = tD[y1 * ND + x1], f = tD[y1 * ND + xp];
        const float2 h = tD[yp * ND + xm], ii = tD[yp * ND + x1], j = tD[yp * ND + xp];
        const float lxx = 0.5f * (kW0 * (c.x - a.x) + kW1 * (f.x - d.x) + kW0 * (j.x - h.x));
        const float lxy = 0.5f * (kW0 * (h.x - a.x) + kW1 * (ii.x - b.x) + kW0 * (j.x - c.x));
        const float lyy = 0.5f * (kW0 * (h.y - a.y) + kW1 * (ii.y - b.y) + kW0 * (j.y - c.y));
        Dout[(size_t)y * g.P + x] = e;
        Lout[(size_t)y * g.P + x] = lxx * lyy - lxy * lxy;
    }
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
    int ty = (g.H + 7) / 8;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_first<<<grid, dim3(32, 8), 0, s>>>(Lt, Lxy, img_stride, g, lt, ty);
}

void launch_hess_det(const float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                     cudaStream_t s) {
    int ty = (g.H + 7) / 8;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_det<<<grid, dim3(32, 8), 0, s>>>(Lxy, Ldet, img_stride, g, lt, ty);
}

void launch_hessian(const float* Lt, float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                    cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_hess_fused<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_hess_fused<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    for (int level = 0; level < lt.n; ++level) {
        const int s = lt.step[level];
        if (s <= 8) {
            const int NL = 32 + 4 * s, ND = 32 + 2 * s;
            const size_t smem = sizeof(float) * (((NL * NL + 3) & ~3) + 2 * ND * ND);
            dim3 grid((g.W + 31) / 32, (g.H + 31) / 32, nimg);
            k_hess_fused<32><<<grid, 256, smem, st>>>(Lt, Lxy, Ldet, img_stride, g, level, s);
        } else {
            const int NL = 64 + 4 * s, ND = 64 + 2 * s;
            const size_t smem = sizeof(float) * (((NL * NL + 3) & ~3) + 2 * ND * ND);
            dim3 grid((g.W + 63) / 64, (g.H + 63) / 64, nimg);
            k_hess_fused<64><<<grid, 1024, smem, st>>>(Lt, Lxy, Ldet, img_stride, g, level, s);
        }
    }
}

void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s) {
    k_component_copy<<<dim3((g.W + 255) / 256, g.H), 256, 0, s>>>(plane, comp, tight, to_tight, g);
}

}  // namespace kz
