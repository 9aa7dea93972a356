// hessian.cu — multiscale derivatives and the scale-normalised Hessian determinant (Eq. 8; A9, A10).
//
// With the dilated Scharr operator at step s (taps at 0, ±s; derivative (−1, 0, 1)/2 after the s-normalisation,
// cross smoothing (3, 10, 3)/16) written N_x, N_y:
//     Lx = N_x L,  Ly = N_y L,  Ldet = N_x(Lx)·N_y(Ly) − N_y(Lx)²
// which equals s⁴(LxxLyy − Lxy²) with per-pixel derivatives (the factor s per derivative order is absorbed in
// N).  Second derivatives read the MATERIALISED first derivatives at clamped coordinates (A10), so they are two
// passes: hess_first (L → Lx, Ly) and hess_det (Lx, Ly → Ldet).  One launch covers every level of every image
// (blockIdx.y packs (level, row-tile)); the per-level step s_i comes from the LevelTable.  (A fused shared-memory
// tile form moving 16 instead of 24 B/px measured slower on B200 at every step: 80-87 µs vs 59 µs per level and
// 4 images — the (T+4s)² halo recomputation costs more than the 8 B/px it saves.)
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

void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s) {
    k_component_copy<<<dim3((g.W + 255) / 256, g.H), 256, 0, s>>>(plane, comp, tight, to_tight, g);
}

}  // namespace kz
