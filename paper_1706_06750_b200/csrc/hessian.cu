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

__global__ void __launch_bounds__(256) k_hess_first(const float* __restrict__ Lt, float* __restrict__ Lx,
                                                    float* __restrict__ Ly, size_t img_stride, Geom g, LevelTable lt,
                                                    int tiles_y) {
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
    Lx[base + (size_t)y * g.P + x] = dx;
    Ly[base + (size_t)y * g.P + x] = dy;
}

__global__ void __launch_bounds__(256) k_hess_det(const float* __restrict__ Lx, const float* __restrict__ Ly,
                                                  float* __restrict__ Ldet, size_t img_stride, Geom g, LevelTable lt,
                                                  int tiles_y) {
    const int level = blockIdx.y / tiles_y, ty = blockIdx.y - level * tiles_y;
    const int x = blockIdx.x * 32 + threadIdx.x, y = ty * 8 + threadIdx.y;
    if (x >= g.W || y >= g.H) return;
    const int s = lt.step[level];
    const size_t base = blockIdx.z * img_stride + (size_t)level * g.plane;
    const float* X = Lx + base;
    const float* Y = Ly + base;
    const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
    const int ym = max(y - s, 0), yp = min(y + s, g.H - 1);
    const size_t om = (size_t)ym * g.P, o0 = (size_t)y * g.P, op = (size_t)yp * g.P;
    // N_x(Lx): x-derivative, smoothing over rows ym, y, yp
    float lxx = 0.5f * (kW0 * (__ldg(X + om + xp) - __ldg(X + om + xm)) + kW1 * (__ldg(X + o0 + xp) - __ldg(X + o0 + xm)) +
                        kW0 * (__ldg(X + op + xp) - __ldg(X + op + xm)));
    // N_y(Lx): y-derivative, smoothing over columns xm, x, xp
    float lxy = 0.5f * (kW0 * (__ldg(X + op + xm) - __ldg(X + om + xm)) + kW1 * (__ldg(X + op + x) - __ldg(X + om + x)) +
                        kW0 * (__ldg(X + op + xp) - __ldg(X + om + xp)));
    // N_y(Ly)
    float lyy = 0.5f * (kW0 * (__ldg(Y + op + xm) - __ldg(Y + om + xm)) + kW1 * (__ldg(Y + op + x) - __ldg(Y + om + x)) +
                        kW0 * (__ldg(Y + op + xp) - __ldg(Y + om + xp)));
    Ldet[base + o0 + x] = lxx * lyy - lxy * lxy;
}

}  // namespace

void launch_hess_first(const float* Lt, float* Lx, float* Ly, size_t img_stride, Geom g, int nimg,
                       const LevelTable& lt, cudaStream_t s) {
    int ty = (g.H + 7) / 8;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_first<<<grid, dim3(32, 8), 0, s>>>(Lt, Lx, Ly, img_stride, g, lt, ty);
}

void launch_hess_det(const float* Lx, const float* Ly, float* Ldet, size_t img_stride, Geom g, int nimg,
                     const LevelTable& lt, cudaStream_t s) {
    int ty = (g.H + 7) / 8;
    dim3 grid((g.W + 31) / 32, ty * lt.n, nimg);
    k_hess_det<<<grid, dim3(32, 8), 0, s>>>(Lx, Ly, Ldet, img_stride, g, lt, ty);
}

}  // namespace kz
