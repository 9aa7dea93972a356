// stencil.cu — Gaussian prefilter, gradient / conductivity and the contrast factor k (sm_100a).
//
//  * prefilter: L0 = G(σ0) * I, separable tile kernel, replicate border (A6, A16).
//  * cond:      c = g(|∇(G(1) * L)|) with ∇ = Scharr step 1 (Eqs. 2-3, A5, A8); one tiled pass
//               computes the σ=1 smoothing at clamped coordinates in shared memory, then the 3x3 Scharr.
//               Mode 0 (level 1) writes |∇|² and the image maximum of |∇| for the k histogram.
//  * khist / kfinal: 300-bin histogram of |∇| over the interior, percentile → k on the device
//               (A7), no host round trip.
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr int TW = 32;  // tile width  (one warp per tile row → coalesced 128 B rows)
constexpr int TH = 16;  // tile height

// -------------------------------------------------------------------------------------------------
// Separable Gaussian over a TW x TH output tile.  The input tile stores I(clamp(u)) for the virtual
// coordinates u of the tile + radius halo, so the separable passes equal the 2-D clamped convolution.
__global__ void __launch_bounds__(256) k_prefilter(const float* __restrict__ in, int64_t in_pitch,
                                                   size_t in_img_stride, float* __restrict__ out,
                                                   size_t out_img_stride, Geom g, GaussTaps t) {
    extern __shared__ float sm[];
    const int R = t.r;
    const int LW = TW + 2 * R, LH = TH + 2 * R;
    float* tin = sm;               // LH x LW
    float* tmid = sm + LH * LW;    // LH x TW
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const float* src = in + blockIdx.z * in_img_stride;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
    for (int i = tid; i < LH * LW; i += nt) {
        int ly = i / LW, lx = i - ly * LW;
        int gx = clampi(x0 - R + lx, 0, g.W - 1), gy = clampi(y0 - R + ly, 0, g.H - 1);
        tin[i] = __ldg(src + (int64_t)gy * in_pitch + gx);
    }
    __syncthreads();
    for (int i = tid; i < LH * TW; i += nt) {
        int ly = i / TW, lx = i - ly * TW;
        const float* row = tin + ly * LW + lx;
        float acc = 0.f;
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(t.w[d], row[d], acc);
        tmid[i] = acc;
    }
    __syncthreads();
    float* dst = out + blockIdx.z * out_img_stride;
    for (int i = tid; i < TH * TW; i += nt) {
        int ly = i / TW, lx = i - ly * TW;
        int x = x0 + lx, y = y0 + ly;
        if (x >= g.W || y >= g.H) continue;
        float acc = 0.f;
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(t.w[d], tmid[(ly + d) * TW + lx], acc);
        dst[(size_t)y * g.P + x] = acc;
    }
}

// -------------------------------------------------------------------------------------------------
// |∇(G1 * L)|² → c (mode 1) or |∇|² + max|∇| (mode 0).  R1 = radius of G(1) (3).
template <int MODE>
__global__ void __launch_bounds__(256) k_cond(const float* __restrict__ L, size_t in_img_stride,
                                              float* __restrict__ out, size_t out_img_stride, Geom g,
                                              GaussTaps t, int diffusivity, const float* __restrict__ kval,
                                              unsigned* __restrict__ hmax_bits) {
    extern __shared__ float sm[];
    const int R = t.r;
    const int H0 = R + 1;                       // halo of the L tile
    const int LW = TW + 2 * H0, LH = TH + 2 * H0;
    const int SW = TW + 2, SH = TH + 2;         // Ls tile: virtual coords [x0-1, x0+TW]
    float* tL = sm;                             // LH x LW : L(clamp(u))
    float* tH = tL + LH * LW;                   // LH x SW : horizontal pass at clamped Ls columns
    float* tS = tH + LH * SW;                   // SH x SW : Ls(clamp(v))
    __shared__ float red[8];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, img = blockIdx.z;
    const float* src = L + img * in_img_stride;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
    for (int i = tid; i < LH * LW; i += nt) {
        int ly = i / LW, lx = i - ly * LW;
        int gx = clampi(x0 - H0 + lx, 0, g.W - 1), gy = clampi(y0 - H0 + ly, 0, g.H - 1);
        tL[i] = __ldg(src + (size_t)gy * g.P + gx);
    }
    __syncthreads();
    // horizontal pass for every L-tile row, at Ls columns v = x0-1+sx, evaluated at clamp(v)
    for (int i = tid; i < LH * SW; i += nt) {
        int ly = i / SW, sx = i - ly * SW;
        int cv = clampi(x0 - 1 + sx, 0, g.W - 1);      // clamped Ls column (image coords)
        int base = cv - (x0 - H0) - R;                 // tile column of cv - R
        const float* row = tL + ly * LW + base;
        float acc = 0.f;
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(t.w[d], row[d], acc);
        tH[i] = acc;
    }
    __syncthreads();
    for (int i = tid; i < SH * SW; i += nt) {
        int sy = i / SW, sx = i - sy * SW;
        int cv = clampi(y0 - 1 + sy, 0, g.H - 1);
        int base = cv - (y0 - H0) - R;
        float acc = 0.f;
        for (int d = 0; d <= 2 * R; ++d) acc = fmaf(t.w[d], tH[(base + d) * SW + sx], acc);
        tS[i] = acc;
    }
    __syncthreads();
    float k2 = 1.f;
    if (MODE == 1) {
        float k = kval[img];
        k2 = k * k;
    }
    float lmax = 0.f;
    float* dst = out + img * out_img_stride;
    for (int i = tid; i < TH * TW; i += nt) {
        int ly = i / TW, lx = i - ly * TW;
        int x = x0 + lx, y = y0 + ly;
        if (x >= g.W || y >= g.H) continue;
        // Ls tile index of virtual coordinate v: v - (x0 - 1); Scharr reads Ls(clamp(x±1), clamp(y+k))
        int xm = clampi(x - 1, 0, g.W - 1) - (x0 - 1), xp = clampi(x + 1, 0, g.W - 1) - (x0 - 1);
        int ym = clampi(y - 1, 0, g.H - 1) - (y0 - 1), yp = clampi(y + 1, 0, g.H - 1) - (y0 - 1);
        int xc = x - (x0 - 1), yc = y - (y0 - 1);
        float gx = 0.1875f * (tS[ym * SW + xp] - tS[ym * SW + xm]) + 0.625f * (tS[yc * SW + xp] - tS[yc * SW + xm]) +
                   0.1875f * (tS[yp * SW + xp] - tS[yp * SW + xm]);
        float gy = 0.1875f * (tS[yp * SW + xm] - tS[ym * SW + xm]) + 0.625f * (tS[yp * SW + xc] - tS[ym * SW + xc]) +
                   0.1875f * (tS[yp * SW + xp] - tS[ym * SW + xp]);
        gx *= 0.5f;
        gy *= 0.5f;
        float g2 = gx * gx + gy * gy;
        if (MODE == 0) {
            dst[(size_t)y * g.P + x] = g2;
            if (x >= 1 && x <= g.W - 2 && y >= 1 && y <= g.H - 2) lmax = fmaxf(lmax, sqrtf(g2));
        } else {
            float q = g2 / k2;
            dst[(size_t)y * g.P + x] = diffusivity == 2 ? 1.f / (1.f + q) : expf(-q);
        }
    }
    if (MODE == 0) {
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if ((tid & 31) == 0) red[tid >> 5] = lmax;
        __syncthreads();
        if (tid == 0) {
            float m = 0.f;
            for (int w = 0; w < nt / 32; ++w) m = fmaxf(m, red[w]);
            atomicMax(hmax_bits + img, __float_as_uint(m));  // non-negative floats order as uints
        }
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
    float q = *p / (k * k);
    *p = diffusivity == 2 ? 1.f / (1.f + q) : expf(-q);
}

}  // namespace

void launch_prefilter(const float* img, int64_t in_pitch, size_t in_img_stride, float* L0, size_t out_img_stride,
                      Geom g, int nimg, const GaussTaps& t, cudaStream_t s) {
    dim3 grid((g.W + TW - 1) / TW, (g.H + TH - 1) / TH, nimg);
    size_t smem = sizeof(float) * ((TH + 2 * t.r) * (TW + 2 * t.r) + (TH + 2 * t.r) * TW);
    k_prefilter<<<grid, dim3(32, 8), smem, s>>>(img, in_pitch, in_img_stride, L0, out_img_stride, g, t);
}

void launch_cond(const float* L, size_t in_img_stride, float* out, size_t out_img_stride, Geom g, int nimg,
                 const GaussTaps& t1, int mode, int diffusivity, const float* kval, unsigned* hmax_bits,
                 cudaStream_t s) {
    dim3 grid((g.W + TW - 1) / TW, (g.H + TH - 1) / TH, nimg);
    const int H0 = t1.r + 1;
    size_t smem = sizeof(float) * ((TH + 2 * H0) * (TW + 2 * H0) + (TH + 2 * H0) * (TW + 2) + (TH + 2) * (TW + 2));
    if (mode == 0)
        k_cond<0><<<grid, dim3(32, 8), smem, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
                                                  hmax_bits);
    else
        k_cond<1><<<grid, dim3(32, 8), smem, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
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
