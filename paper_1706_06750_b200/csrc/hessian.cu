// hessian.cu — multiscale derivatives and the scale-normalised Hessian determinant (Eq. 8; A9, A10).
//
// With the dilated Scharr operator at step s (taps at 0, ±s; derivative (−1, 0, 1)/2 after the s-normalisation,
// cross smoothing (3, 10, 3)/16) written N_x, N_y:
//     Lx = N_x L,  Ly = N_y L,  Ldet = N_x(Lx)·N_y(Ly) − N_y(Lx)²
// which equals s⁴(LxxLyy − Lxy²) with per-pixel derivatives (the factor s per derivative order is absorbed in
// N).  Second derivatives read the MATERIALISED first derivatives at clamped coordinates (A10), so they are two
// passes: hess_first (L → Lx, Ly) and hess_det (Lx, Ly → Ldet).  One launch covers every level of every image
// (blockIdx.z packs (image, level), blockIdx.y the chain block); the per-level step s_i comes from the LevelTable.  (A fused shared-memory
// tile form moving 16 instead of 24 B/px measured slower on B200 at every step: 80-87 µs vs 59 µs per level and
// 4 images — the (T+4s)² halo recomputation costs more than the 8 B/px it saves.)
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr float kW0 = 0.1875f, kW1 = 0.625f;  // (3, 10, 3) / 16

__device__ __forceinline__ float det_from_ring(float2 a, float2 b, float2 c, float2 d, float2 f, float2 h, float2 i,
                                               float2 j) {
    const float lxx = 0.5f * (kW0 * (c.x - a.x) + kW1 * (f.x - d.x) + kW0 * (j.x - h.x));  // N_x(Lx)
    const float lxy = 0.5f * (kW0 * (h.x - a.x) + kW1 * (i.x - b.x) + kW0 * (j.x - c.x));  // N_y(Lx)
    const float lyy = 0.5f * (kW0 * (h.y - a.y) + kW1 * (i.y - b.y) + kW0 * (j.y - c.y));  // N_y(Ly)
    return lxx * lyy - lxy * lxy;
}

// Chain form: a thread computes R outputs of one column at rows y_j = y_0 + j·s (j < R) — a "chain" in the row
// residue class of y_0 mod s.  Output j reads rows y_j − s, y_j, y_j + s = chain rows j−1, j, j+1, so the R outputs
// need (R + 2) rows × 3 taps instead of 8R taps: 44% fewer L1 wavefronts at R = 4, 61% at R = 8.  Chains tile the
// rows band by band: band b = [b·R·s, (b+1)·R·s) holds the s chains y_0 = b·R·s + r, r < s.  Every tap is read at
// clamped coordinates (A10/A16); the clamp of row y_j ± s equals the clamp of the neighbouring chain row.
constexpr int kChainR = 8;  // measured at 1920x1200 (256-image step): R = 8 51.3 ms, 12 53.0, 4 61.1, 32x32 tiles 59.2

// Chains of one level: s per band, ceil(H / (R·s)) bands.  grid.y covers the largest level; blocks past a level's
// chain count exit at once.  b = ch / s via a float quotient: (ch + ½)/s stays >= 1/(2s) away from an integer, far
// beyond the error of __fdividef at these sizes (ch < 2^16, s < 64).
__device__ __forceinline__ int chain_band(int ch, int s) { return (int)__fdividef((float)ch + 0.5f, (float)s); }

// Interior chains (every tap row and column inside the image — all but the border warps) take a clamp-free path
// with the step s as a compile-time constant: one row pointer per chain row and the x − s, x, x + s taps as
// immediate offsets from it (~4 instructions per 3 loads instead of ~10).  Border chains and steps above
// kMaxTemplStep use the clamped generic path.  (The kernels dispatch on s per CTA; s is uniform per level.)
constexpr int kMaxTemplStep = 24;

template <int R, int SC, class T>
__device__ __forceinline__ bool chain_setup(Geom g, int s_rt, int ch, int x, int& s, int& y0, bool& fast) {
    s = SC > 0 ? SC : s_rt;
    const int nch = s * ((g.H + R * s - 1) / (R * s));
    if (ch >= nch || x >= g.W) return false;
    const int b = SC > 0 ? ch / SC : chain_band(ch, s);
    y0 = b * R * s + (ch - b * s);
    fast = SC > 0 && y0 >= s && y0 + R * s <= g.H - 1 && x >= s && x + s <= g.W - 1;
    return true;
}

// Loads columns x−s, x, x+s of chain rows −1..R (rows y0 + (k−1)s, clamped on the generic path).
template <int R, int SC, class T>
__device__ __forceinline__ void chain_load(const T* __restrict__ src, Geom g, int s, int y0, int x, bool fast,
                                           T (&a)[R + 2], T (&m)[R + 2], T (&c)[R + 2]) {
    if (SC > 0 && fast) {
#pragma unroll
        for (int k = 0; k < R + 2; ++k) {
            const T* p = src + (unsigned)((y0 + (k - 1) * SC) * g.P + x);
            a[k] = __ldg(p - SC);
            m[k] = __ldg(p);
            c[k] = __ldg(p + SC);
        }
    } else {
        const int xm = max(x - s, 0), xp = min(x + s, g.W - 1);
#pragma unroll
        for (int k = 0; k < R + 2; ++k) {
            const int ro = clampi(y0 + (k - 1) * s, 0, g.H - 1) * g.P;
            a[k] = __ldg(src + (unsigned)(ro + xm));  // unsigned 32-bit offsets: one IMAD.WIDE.U32 per address
            m[k] = __ldg(src + (unsigned)(ro + x));
            c[k] = __ldg(src + (unsigned)(ro + xp));
        }
    }
}

template <int R, int SC>
__device__ __forceinline__ void hess_first_body(const float* __restrict__ L, float2* __restrict__ D, Geom g, int s_rt,
                                                int ch, int x) {
    int s, y0;
    bool fast;
    if (!chain_setup<R, SC, float>(g, s_rt, ch, x, s, y0, fast)) return;
    float a[R + 2], m[R + 2], c[R + 2];  // columns x−s, x, x+s of chain rows −1..R
    chain_load<R, SC, float>(L, g, s, y0, x, fast, a, m, c);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int y = y0 + j * s;
        const float2 v = make_float2(0.5f * (kW0 * (c[j] - a[j]) + kW1 * (c[j + 1] - a[j + 1]) + kW0 * (c[j + 2] - a[j + 2])),
                                     0.5f * (kW0 * (a[j + 2] - a[j]) + kW1 * (m[j + 2] - m[j]) + kW0 * (c[j + 2] - c[j])));
        if (fast || y < g.H) __stwb(D + (unsigned)(y * g.P + x), v);
    }
}

template <int R, int SC>
__device__ __forceinline__ void hess_det_body(const float2* __restrict__ D, float* __restrict__ O, Geom g, int s_rt,
                                              int ch, int x) {
    int s, y0;
    bool fast;
    if (!chain_setup<R, SC, float2>(g, s_rt, ch, x, s, y0, fast)) return;
    float2 a[R + 2], m[R + 2], c[R + 2];
    chain_load<R, SC, float2>(D, g, s, y0, x, fast, a, m, c);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int y = y0 + j * s;
        const float v = det_from_ring(a[j], m[j], c[j], a[j + 1], c[j + 1], a[j + 2], m[j + 2], c[j + 2]);
        if (fast || y < g.H) __stwb(O + (unsigned)(y * g.P + x), v);
    }
}

#define KZ_STEP_CASES(F) \
    F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14) F(15) F(16) F(17) F(18) F(19) F(20) \
    F(21) F(22) F(23) F(24)

template <int R>
__global__ void __launch_bounds__(256) k_hess_first_chain(const float* __restrict__ Lt, float2* __restrict__ Lxy,
                                                          size_t img_stride, Geom g, LevelTable lt) {
    const int img = chain_band(blockIdx.z, lt.n), level = blockIdx.z - img * lt.n;
    const int s = lt.step[level];
    const int ch = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const size_t base = img * img_stride + (size_t)level * g.plane;
    const float* L = opaque(Lt + base);
    float2* D = opaque(Lxy + base);
    switch (s) {
#define KZ_CASE(S) \
    case S: hess_first_body<R, S>(L, D, g, s, ch, x); break;
        KZ_STEP_CASES(KZ_CASE)
#undef KZ_CASE
        default: hess_first_body<R, 0>(L, D, g, s, ch, x); break;
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_hess_det_chain(const float2* __restrict__ Lxy, float* __restrict__ Ldet,
                                                        size_t img_stride, Geom g, LevelTable lt) {
    const int img = chain_band(blockIdx.z, lt.n), level = blockIdx.z - img * lt.n;
    const int s = lt.step[level];
    const int ch = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const size_t base = img * img_stride + (size_t)level * g.plane;
    const float2* D = opaque(Lxy + base);
    float* O = opaque(Ldet + base);
    switch (s) {
#define KZ_CASE(S) \
    case S: hess_det_body<R, S>(D, O, g, s, ch, x); break;
        KZ_STEP_CASES(KZ_CASE)
#undef KZ_CASE
        default: hess_det_body<R, 0>(D, O, g, s, ch, x); break;
    }
}

template <int R>
int max_chain_blocks(Geom g, const LevelTable& lt) {
    int m = 1;
    for (int l = 0; l < lt.n; ++l) {
        const int s = lt.step[l];
        m = max(m, (s * ((g.H + R * s - 1) / (R * s)) + 7) / 8);
    }
    return m;
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
    const dim3 grid((g.W + 31) / 32, max_chain_blocks<kChainR>(g, lt), nimg * lt.n);
    k_hess_first_chain<kChainR><<<grid, dim3(32, 8), 0, s>>>(Lt, Lxy, img_stride, g, lt);
}

void launch_hess_det(const float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                     cudaStream_t s) {
    const dim3 grid((g.W + 31) / 32, max_chain_blocks<kChainR>(g, lt), nimg * lt.n);
    k_hess_det_chain<kChainR><<<grid, dim3(32, 8), 0, s>>>(Lxy, Ldet, img_stride, g, lt);
}

void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s) {
    k_component_copy<<<dim3((g.W + 255) / 256, g.H), 256, 0, s>>>(plane, comp, tight, to_tight, g);
}

}  // namespace kz
