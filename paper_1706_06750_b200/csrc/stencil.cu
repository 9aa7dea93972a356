// stencil.cu — Gaussian prefilter, gradient / conductivity and the contrast factor k (sm_100a).
//
//  * prefilter: L0 = G(σ0) * I, separable tile kernel, replicate border (A6, A16).
//  * cond:      c = g(|∇(G(1) * L)|) with ∇ = Scharr step 1 (Eqs. 2-3, A5, A8); one warp-streaming
//               pass computes the σ=1 smoothing at clamped coordinates in registers, then the 3x3 Scharr.
//               Mode 0 (level 1) writes |∇|² and the image maximum of |∇| for the k histogram.
//  * khist / kfinal: 300-bin histogram of |∇| over the interior, percentile → k on the device
//               (A7), no host round trip.
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr int TW = 32;  // tile width  (one warp per tile row → coalesced 128 B rows)
constexpr int TH = 32;  // tile height (block 32 x 8, four output rows per thread)

__device__ __forceinline__ float frcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// -------------------------------------------------------------------------------------------------
// Separable Gaussian over a TW x TH output tile.  The input tile stores I(clamp(u)) for the virtual
// coordinates u of the tile + radius halo, so the separable passes equal the 2-D clamped convolution.
template <int R>
__global__ void __launch_bounds__(256) k_prefilter(const float* __restrict__ in, int64_t in_pitch,
                                                   size_t in_img_stride, float* __restrict__ out,
                                                   size_t out_img_stride, Geom g, GaussTaps t) {
    constexpr int LW = TW + 2 * R, LH = TH + 2 * R;
    __shared__ float tin[LH][LW];
    __shared__ float tmid[LH][TW];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const float* src = in + blockIdx.z * in_img_stride;
    const int tx = threadIdx.x, ty = threadIdx.y;
    {   // all tile loads issued before any shared store
        constexpr int KR = (LH + 7) / 8, KC = (LW + 31) / 32;
        float v[KR][KC];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int ly = ty + 8 * k;
            const float* row = src + (int64_t)clampi(y0 - R + ly, 0, g.H - 1) * in_pitch;
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int lx = tx + 32 * j;
                v[k][j] = (ly < LH && lx < LW) ? __ldg(row + clampi(x0 - R + lx, 0, g.W - 1)) : 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k)
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int ly = ty + 8 * k, lx = tx + 32 * j;
                if (ly < LH && lx < LW) tin[ly][lx] = v[k][j];
            }
    }
    float w[2 * R + 1];
#pragma unroll
    for (int d = 0; d <= 2 * R; ++d) w[d] = t.w[d];
    __syncthreads();
    for (int ly = ty; ly < LH; ly += 8) {
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(w[d], tin[ly][tx + d], acc);
        tmid[ly][tx] = acc;
    }
    __syncthreads();
    float* dst = out + blockIdx.z * out_img_stride;
    const int x = x0 + tx;
#pragma unroll
    for (int k = 0; k < TH / 8; ++k) {
        const int ly = ty + 8 * k, y = y0 + ly;
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(w[d], tmid[ly + d][tx], acc);
        if (x < g.W && y < g.H) dst[(size_t)y * g.P + x] = acc;
    }
}

// G(σ=1) has radius 3 (A6).
constexpr int R1 = 3;

// -------------------------------------------------------------------------------------------------
// |∇(G1 * L)|² → c (mode 1) or |∇|² + max|∇| (mode 0), warp-streaming: a warp owns 30 output columns — lane l holds the
// Ls column x0-1+l, so lanes 1..30 produce outputs and lanes 0 / 31 are the Ls halo — and walks CS_SEG output rows
// top to bottom.  Per input row it loads the 38-column L segment (clamped) into a per-warp shared row, forms the
// horizontal G1 for its column, keeps the last 7 horizontal results in registers for the vertical G1, keeps the
// last 3 Ls rows for the Scharr, and reads the Ls of its neighbour columns with shuffles.  Every L value is read
// from HBM ~1.1 times; ~50 instructions per 30 pixels per row.  Border semantics (A16): Ls is evaluated at clamped
// coordinates (its window rows/columns are L at clamped indices), and the Scharr reads Ls at clamp(x±1),
// clamp(y±1) — the column-neighbour and first/last-row selects below.
constexpr int CS_SEG = 64;

template <int MODE>
__global__ void __launch_bounds__(256) k_cond_stream(const float* __restrict__ L, size_t in_img_stride,
                                                     float* __restrict__ out, size_t out_img_stride, Geom g,
                                                     GaussTaps t, int diffusivity, const float* __restrict__ kval,
                                                     unsigned* __restrict__ hmax_bits) {
    __shared__ float rowbuf[8][2][40];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 8 + warp) * 30;
    if (x0 >= g.W) return;  // warp-uniform
    const int y0 = blockIdx.y * CS_SEG, img = blockIdx.z;
    const float* src = L + img * in_img_stride;
    const int W = g.W, H = g.H;
    const int xcol = x0 - 1 + lane;                   // this lane's Ls column (virtual)
    const int hb = clampi(xcol, 0, W - 1) - (x0 - 4) - R1;  // row-buffer index of tap d = -3
    const int gxa = clampi(x0 - 4 + lane, 0, W - 1), gxb = clampi(x0 + 28 + lane, 0, W - 1);
    float w[2 * R1 + 1];
#pragma unroll
    for (int d = 0; d <= 2 * R1; ++d) w[d] = t.w[d];
    float ik2 = 1.f;
    if (MODE == 1) {
        const float k = kval[img];
        ik2 = frcp(k * k);
    }
    float hw[2 * R1 + 1];
#pragma unroll
    for (int d = 0; d <= 2 * R1; ++d) hw[d] = 0.f;
    float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, lmax = 0.f;
    float* dst = out + img * out_img_stride;
    const bool outcol = lane >= 1 && lane <= 30 && xcol < W;
    const bool at_left = xcol == 0, at_right = xcol == W - 1;
    const int u0 = y0 - 4, u1 = y0 + CS_SEG + 3;
    // software pipeline: the next row's two loads are in flight while the current row is processed
    const float* r0 = src + (size_t)clampi(u0, 0, H - 1) * g.P;
    float na = __ldg(r0 + gxa), nb = lane < 6 ? __ldg(r0 + gxb) : 0.f;
    int buf = 0;
    for (int u = u0; u <= u1; ++u) {
        rowbuf[warp][buf][lane] = na;
        if (lane < 6) rowbuf[warp][buf][32 + lane] = nb;
        if (u < u1) {
            const float* rn = src + (size_t)clampi(u + 1, 0, H - 1) * g.P;
            na = __ldg(rn + gxa);
            nb = lane < 6 ? __ldg(rn + gxb) : 0.f;
        }
        __syncwarp();
        float hh = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R1; ++d) hh = fmaf(w[d], rowbuf[warp][buf][hb + d], hh);
        buf ^= 1;  // the other buffer is refilled next iteration; this one is not written again until then
#pragma unroll
        for (int d = 0; d < 2 * R1; ++d) hw[d] = hw[d + 1];
        hw[2 * R1] = hh;
        if (u < y0 + 2) continue;  // window rows u-6..u not yet complete for Ls(u-3), v >= y0-1
        float lsv = 0.f;
#pragma unroll
        for (int d = 0; d <= 2 * R1; ++d) lsv = fmaf(w[d], hw[d], lsv);
        ls0 = ls1;
        ls1 = ls2;
        ls2 = lsv;
        if (u < y0 + 4) continue;
        const int y = u - 4;
        if (y >= H) break;
        const float lm = (y == 0) ? ls1 : ls0, lp = (y == H - 1) ? ls1 : ls2;
        // vertical (3,10,3)/16 smoothing and vertical difference of this column, neighbours by shuffles
        const float sv = 0.1875f * lm + 0.625f * ls1 + 0.1875f * lp;
        const float dv = lp - lm;
        float svl = __shfl_up_sync(0xffffffffu, sv, 1), svr = __shfl_down_sync(0xffffffffu, sv, 1);
        float dvl = __shfl_up_sync(0xffffffffu, dv, 1), dvr = __shfl_down_sync(0xffffffffu, dv, 1);
        if (at_left) { svl = sv; dvl = dv; }
        if (at_right) { svr = sv; dvr = dv; }
        const float gx = 0.5f * (svr - svl);
        const float gy = 0.5f * (0.1875f * dvl + 0.625f * dv + 0.1875f * dvr);
        const float g2 = gx * gx + gy * gy;
        if (outcol) {
            if (MODE == 0) {
                dst[(size_t)y * g.P + xcol] = g2;
                if (xcol >= 1 && xcol <= W - 2 && y >= 1 && y <= H - 2) lmax = fmaxf(lmax, sqrtf(g2));
            } else {
                const float q = g2 * ik2;
                dst[(size_t)y * g.P + xcol] = diffusivity == 2 ? frcp(1.f + q) : __expf(-q);
            }
        }
    }
    if (MODE == 0) {
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if (lane == 0) atomicMax(hmax_bits + img, __float_as_uint(lmax));
    }
}

// -------------------------------------------------------------------------------------------------
// Histogram of |∇| over the interior (A7): warp-aggregated shared-memory atomics, one global add per bin.
__global__ void __launch_bounds__(256) k_khist(const float* __restrict__ g2buf, size_t img_stride, Geom g, int bins,
                                               const unsigned* __restrict__ hmax_bits, int* __restrict__ hist) {
    extern __shared__ int sh[];
    const int img = blockIdx.y;
    for (int i = threadIdx.x; i < bins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const float hmax = __uint_as_float(hmax_bits[img]);
    const float fb = (float)bins;
    const float* src = g2buf + img * img_stride;
    const int iw = g.W - 2, ih = g.H - 2;
    const long long total = (long long)iw * ih;
    const unsigned lane = threadIdx.x & 31;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < total; base += (long long)gridDim.x * blockDim.x) {
        long long i = base + threadIdx.x;
        int b = -1;
        if (i < total) {
            int y = 1 + (int)(i / iw), x = 1 + (int)(i % iw);
            float gm = sqrtf(src[(size_t)y * g.P + x]);
            if (gm > 0.f) b = min((int)floorf(fb * gm / hmax), bins - 1);
        }
        unsigned peers = __match_any_sync(0xffffffffu, b);
        int leader = __ffs(peers) - 1;
        if (b >= 0 && (int)lane == leader) atomicAdd(&sh[b], __popc(peers));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[img * bins + i], sh[i]);
}

// Percentile → k = hmax·(b+1)/bins with b the first bin whose cumulative count reaches floor(perc·n).
__global__ void k_kfinal(const int* __restrict__ hist, int bins, const unsigned* __restrict__ hmax_bits,
                         double perc, double k_override, float* __restrict__ kval, int* __restrict__ fallback) {
    const int img = blockIdx.x;
    if (threadIdx.x != 0) return;
    if (k_override > 0) {
        kval[img] = (float)k_override;
        fallback[img] = 0;
        return;
    }
    const int* h = hist + img * bins;
    long long n = 0;
    for (int b = 0; b < bins; ++b) n += h[b];
    if (n == 0) {
        kval[img] = 0.03f;
        fallback[img] = 1;
        return;
    }
    long long thr = (long long)floor(perc * (double)n);
    long long cum = 0;
    int b = 0;
    for (b = 0; b < bins; ++b) {
        cum += h[b];
        if (cum >= thr) break;
    }
    if (b >= bins) b = bins - 1;
    kval[img] = (float)((double)__uint_as_float(hmax_bits[img]) * (double)(b + 1) / (double)bins);
    fallback[img] = 0;
}

__global__ void __launch_bounds__(256) k_c_from_g2(float* __restrict__ buf, size_t img_stride, Geom g,
                                                   int diffusivity, const float* __restrict__ kval) {
    const int img = blockIdx.z;
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= g.W) return;
    float k = kval[img];
    float* p = buf + img * img_stride + (size_t)y * g.P + x;
    const float q = *p * frcp(k * k);
    *p = diffusivity == 2 ? frcp(1.f + q) : __expf(-q);
}

}  // namespace

void launch_prefilter(const float* img, int64_t in_pitch, size_t in_img_stride, float* L0, size_t out_img_stride,
                      Geom g, int nimg, const GaussTaps& t, cudaStream_t s) {
    dim3 grid((g.W + TW - 1) / TW, (g.H + TH - 1) / TH, nimg);
    dim3 block(32, 8);
    switch (t.r) {
#define KZ_PF(R) \
    case R: k_prefilter<R><<<grid, block, 0, s>>>(img, in_pitch, in_img_stride, L0, out_img_stride, g, t); break;
        KZ_PF(1) KZ_PF(2) KZ_PF(3) KZ_PF(4) KZ_PF(5) KZ_PF(6) KZ_PF(7) KZ_PF(8) KZ_PF(9) KZ_PF(10) KZ_PF(11)
        KZ_PF(12) KZ_PF(13) KZ_PF(14) KZ_PF(15) KZ_PF(16) KZ_PF(17) KZ_PF(18) KZ_PF(19) KZ_PF(20) KZ_PF(21)
        KZ_PF(22) KZ_PF(23) KZ_PF(24)
#undef KZ_PF
        default: break;
    }
}

void launch_cond(const float* L, size_t in_img_stride, float* out, size_t out_img_stride, Geom g, int nimg,
                 const GaussTaps& t1, int mode, int diffusivity, const float* kval, unsigned* hmax_bits,
                 cudaStream_t s) {
    const int strips = (g.W + 29) / 30;
    dim3 grid((strips + 7) / 8, (g.H + CS_SEG - 1) / CS_SEG, nimg);
    if (mode == 0)
        k_cond_stream<0><<<grid, 256, 0, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
                                              hmax_bits);
    else
        k_cond_stream<1><<<grid, 256, 0, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
                                              hmax_bits);
}

void launch_khist(const float* g2, size_t img_stride, Geom g, int nimg, int bins, const unsigned* hmax_bits, int* hist,
                  cudaStream_t s) {
    long long total = (long long)(g.W - 2) * (g.H - 2);
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148) blocks = 148;
    k_khist<<<dim3(blocks, nimg), 256, sizeof(int) * bins, s>>>(g2, img_stride, g, bins, hmax_bits, hist);
}

void launch_kfinal(const int* hist, int bins, const unsigned* hmax_bits, int nimg, double perc, double k_override,
                   float* kval, int* fallback, cudaStream_t s) {
    k_kfinal<<<nimg, 32, 0, s>>>(hist, bins, hmax_bits, perc, k_override, kval, fallback);
}

void launch_c_from_g2(float* buf, size_t img_stride, Geom g, int nimg, int diffusivity, const float* kval,
                      cudaStream_t s) {
    dim3 grid((g.W + 255) / 256, g.H, nimg);
    k_c_from_g2<<<grid, 256, 0, s>>>(buf, img_stride, g, diffusivity, kval);
}

}  // namespace kz
