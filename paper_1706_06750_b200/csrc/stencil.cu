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

// -------------------------------------------------------------------------------------------------
// |∇(G1 * L)|² → c (mode 1) or |∇|² + max|∇| (mode 0).  G(σ=1) has radius 3 (A6).
// Shared-memory traffic is kept to ~12 accesses per pixel with register sliding windows:
//   L tile  tL[u]  = L(clamp(u)) for u in [x0-4, x0+35]²   (odd pitch 41: per-row sweeps are conflict free)
//   tH[r][v]       = Σ_d g_d tL[r][v+d]      horizontal G1, one thread per tile row (two halves)
//   tS[v][v']      = Σ_d g_d tH[v+d][v']     vertical G1, one thread per column (four row groups)
// tS holds Ls at the virtual coordinates [x0-1, x0+32]²; it equals Ls(clamp(v)) wherever v is inside the
// image, and the Scharr reads Ls at clamped coordinates only (A16), so border tiles need no special path.
constexpr int R1 = 3;
template <int MODE>
__global__ void __launch_bounds__(256) k_cond(const float* __restrict__ L, size_t in_img_stride,
                                              float* __restrict__ out, size_t out_img_stride, Geom g,
                                              GaussTaps t, int diffusivity, const float* __restrict__ kval,
                                              unsigned* __restrict__ hmax_bits) {
    constexpr int H0 = R1 + 1;              // halo of the L tile
    constexpr int LN = TW + 2 * H0;         // 40 (square tile, TW == TH)
    constexpr int SN = TW + 2;              // 34
    __shared__ float tL[LN][LN + 1];
    __shared__ float tH[LN][SN + 1];
    __shared__ float tS[SN][SN + 1];
    __shared__ float red[8];
    static_assert(TW == TH, "square tiles");
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, img = blockIdx.z;
    const float* src = L + img * in_img_stride;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    {   // all tile loads issued before any shared store (LN = 40 rows: 5 per warp; 40 columns: 32 + 8 lanes)
        constexpr int KR = LN / 8;
        const int gx0 = clampi(x0 - H0 + tx, 0, g.W - 1), gx1 = clampi(x0 - H0 + 32 + tx, 0, g.W - 1);
        float v0[KR], v1[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const float* row = src + (size_t)clampi(y0 - H0 + ty + 8 * k, 0, g.H - 1) * g.P;
            v0[k] = __ldg(row + gx0);
            v1[k] = tx < LN - 32 ? __ldg(row + gx1) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            tL[ty + 8 * k][tx] = v0[k];
            if (tx < LN - 32) tL[ty + 8 * k][32 + tx] = v1[k];
        }
    }
    float w[2 * R1 + 1];
#pragma unroll
    for (int d = 0; d <= 2 * R1; ++d) w[d] = t.w[d];
    __syncthreads();
    if (tid < 2 * LN) {  // horizontal: row r, output columns [17h, 17h+17)
        constexpr int NO = SN / 2;  // 17
        const int r = tid % LN, h = tid / LN;
        float win[NO + 2 * R1];
#pragma unroll
        for (int i = 0; i < NO + 2 * R1; ++i) win[i] = tL[r][NO * h + i];
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            float acc = 0.f;
#pragma unroll
            for (int d = 0; d <= 2 * R1; ++d) acc = fmaf(w[d], win[o + d], acc);
            tH[r][NO * h + o] = acc;
        }
    }
    __syncthreads();
    if (tid < 4 * SN) {  // vertical: column v, output rows [9q, min(9q+9, 34))
        constexpr int NO = 9;
        const int v = tid % SN, q = tid / SN;
        const int r0 = NO * q;
        float win[NO + 2 * R1];
#pragma unroll
        for (int i = 0; i < NO + 2 * R1; ++i) win[i] = (r0 + i < LN) ? tH[r0 + i][v] : 0.f;
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            if (r0 + o < SN) {
                float acc = 0.f;
#pragma unroll
                for (int d = 0; d <= 2 * R1; ++d) acc = fmaf(w[d], win[o + d], acc);
                tS[r0 + o][v] = acc;
            }
        }
    }
    __syncthreads();
    float ik2 = 1.f;
    if (MODE == 1) {
        const float k = kval[img];
        ik2 = frcp(k * k);
    }
    float lmax = 0.f;
    float* dst = out + img * out_img_stride;
    const int x = x0 + tx;
    // tS index of virtual coordinate v is v - (x0 - 1); the Scharr reads Ls(clamp(x±1), clamp(y±1))
    const int xm = clampi(x - 1, 0, g.W - 1) - (x0 - 1), xp = clampi(x + 1, 0, g.W - 1) - (x0 - 1), xc = tx + 1;
    const int yb = y0 + 4 * ty;  // four output rows per thread
    float cm[6], cc[6], cp[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const int yy = clampi(yb - 1 + i, 0, g.H - 1) - (y0 - 1);
        cm[i] = tS[yy][xm];
        cc[i] = tS[yy][xc];
        cp[i] = tS[yy][xp];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int y = yb + k;
        // window rows k, k+1, k+2 hold clamp(y-1), y, clamp(y+1) unless y is the first/last image row
        const bool top = (y == 0), bot = (y == g.H - 1);
        const float mm = top ? cm[k + 1] : cm[k], mc = top ? cc[k + 1] : cc[k], mp = top ? cp[k + 1] : cp[k];
        const float pm = bot ? cm[k + 1] : cm[k + 2], pc = bot ? cc[k + 1] : cc[k + 2], pp = bot ? cp[k + 1] : cp[k + 2];
        float gx = 0.1875f * (mp - mm) + 0.625f * (cp[k + 1] - cm[k + 1]) + 0.1875f * (pp - pm);
        float gy = 0.1875f * (pm - mm) + 0.625f * (pc - mc) + 0.1875f * (pp - mp);
        gx *= 0.5f;
        gy *= 0.5f;
        const float g2 = gx * gx + gy * gy;
        if (x < g.W && y < g.H) {
            if (MODE == 0) {
                dst[(size_t)y * g.P + x] = g2;
                if (x >= 1 && x <= g.W - 2 && y >= 1 && y <= g.H - 2) lmax = fmaxf(lmax, sqrtf(g2));
            } else {
                const float q = g2 * ik2;
                dst[(size_t)y * g.P + x] = diffusivity == 2 ? frcp(1.f + q) : __expf(-q);
            }
        }
    }
    if (MODE == 0) {
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if (tx == 0) red[ty] = lmax;
        __syncthreads();
        if (tid == 0) {
            float m = 0.f;
            for (int wv = 0; wv < 8; ++wv) m = fmaxf(m, red[wv]);
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
    dim3 grid((g.W + TW - 1) / TW, (g.H + TH - 1) / TH, nimg);
    if (mode == 0)
        k_cond<0><<<grid, dim3(32, 8), 0, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
                                               hmax_bits);
    else
        k_cond<1><<<grid, dim3(32, 8), 0, s>>>(L, in_img_stride, out, out_img_stride, g, t1, diffusivity, kval,
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
