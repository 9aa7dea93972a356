// describe.cu — dominant orientation (A14) and 64-D M-SURF (A15).
//
// One warp per keypoint over the FLAT list of all keypoints of all levels and images (the paper's load-balancing
// remedy: "all the image scales are computed at the same time"), persistent grid of one full wave (occupancy-sized).
//   orientation: 113 samples at kp + σ(u, v), u² + v² <= 36, spread over the lanes; Gaussian weight
//                exp(−(u²+v²)/12.5) (std 2.5σ); the weighted (Lx, Ly) vectors go to shared memory; lanes own the
//                window centres θ_k = 2πk/nwin and sum the vectors within ±π/6; a warp arg-max (first k on
//                ties) picks the longest sum; angle = atan2 of it in [0, 2π).
//   M-SURF:      24 x 24 samples at step σ rotated by the angle, bilinear (Lx, Ly) rotated into the keypoint
//                frame (du, dv) and staged in shared memory; lane pair (2·sr, 2·sr+1) accumulates subregion sr's 9 x 9
//                window (Gaussian std 2.5 about its centre), the 4x4 mask (std 1.5) weights it, the warp
//                normalises the 64-vector and writes it with 16-byte stores.
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr int kOriSamples = 113;
__constant__ float c_ori_u[kOriSamples], c_ori_v[kOriSamples], c_ori_w[kOriSamples];
__constant__ float c_w1[81];  // exp(-((i-4)^2 + (j-4)^2) / (2 * 2.5^2)), i, j = 0..8
__constant__ float c_w2[16];  // exp(-((a-1.5)^2 + (b-1.5)^2) / (2 * 1.5^2)), index 4b + a

constexpr float kTwoPi = 6.283185307179586f;
constexpr float kPi = 3.141592653589793f;

// Bilinear (Lx, Ly) at (px, py) with clamped taps (A14, A16): four 8-byte loads of the interleaved plane.
__device__ __forceinline__ float2 bilinear2(const float2* __restrict__ img, int W, int H, int P, float px, float py) {
    const float fx0 = floorf(px), fy0 = floorf(py);
    const float fx = px - fx0, fy = py - fy0;
    const int x0 = (int)fx0, y0 = (int)fy0;
    const int xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
    const int ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
    const float2 v00 = __ldg(img + (size_t)ya * P + xa), v10 = __ldg(img + (size_t)ya * P + xb);
    const float2 v01 = __ldg(img + (size_t)yb * P + xa), v11 = __ldg(img + (size_t)yb * P + xb);
    return make_float2((1.f - fy) * ((1.f - fx) * v00.x + fx * v10.x) + fy * ((1.f - fx) * v01.x + fx * v11.x),
                       (1.f - fy) * ((1.f - fx) * v00.y + fx * v10.y) + fy * ((1.f - fx) * v01.y + fx * v11.y));
}

constexpr int kWarps = 8;
constexpr int kSP = 25;         // pitch of the staged 24 x 24 M-SURF samples
constexpr int kMaxBinWin = 48;  // binned orientation path: nwin % 6 == 0 and nwin <= 48 (2·nwin <= 96 bins)

__global__ void __launch_bounds__(256) k_describe(const float2* __restrict__ Lxy,
                                                  const cudaTextureObject_t* __restrict__ texs, size_t img_stride, Geom g, int nimg, kaze_keypoint* __restrict__ kps,
                                                  const int* __restrict__ counts, int cap, float* __restrict__ desc,
                                                  int nwin, int keep_angle, int N) {
    __shared__ int pre[kMaxBatch + 1];
    __shared__ __align__(16) float sbuf[kWarps][2 * kSP * 24];
    if (threadIdx.x == 0) {
        int r = 0;
        for (int i = 0; i < nimg; ++i) {
            pre[i] = r;
            r += min(max(counts[i], 0), cap);
        }
        pre[nimg] = r;
    }
    __syncthreads();
    const int total = pre[nimg];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sx = sbuf[warp];
    float* sy = sx + kSP * 24;
    for (int f = blockIdx.x * kWarps + warp; f < total; f += gridDim.x * kWarps) {
        int img = 0;
        while (img + 1 < nimg && pre[img + 1] <= f) ++img;  // nimg is small
        const int k = f - pre[img];
        kaze_keypoint* kp = kps + (size_t)img * cap + k;
        const float x = kp->x, y = kp->y, sigma = kp->sigma;
        const int level = kp->level;
        const float2* lxy = Lxy + img * img_stride + (size_t)level * g.plane;
        const cudaTextureObject_t tex = texs[img * N + level];
        float angle;
        int flags = 0;
        if (keep_angle) {
            angle = kp->angle;
        } else {
            // ---- orientation ----
            float best = 0.f, bx = 0.f, by = 0.f;
            int bk = 0x7fffffff;
            if (nwin % 6 == 0 && nwin <= kMaxBinWin) {
                // Fine angular bins of width π/nwin: window k (centre 2πk/nwin, half-width π/6) is exactly the bins
                // [2k − h, 2k + h), h = nwin/6, up to the measure-zero boundary points.  A stable counting sort
                // (integer counts; ranks from __match_any_sync, so the order is deterministic) groups the samples by
                // bin, each bin is summed in sample order, and each window sums its 2h bins in bin order: ~500
                // instructions per keypoint instead of a 113 x nwin scan.
                const int nb = 2 * nwin, h = nwin / 6;
                int* cnt = reinterpret_cast<int*>(sx);           // [nb]
                int* off = cnt + kMaxBinWin * 2;                 // [nb]
                float2* srt = reinterpret_cast<float2*>(off + kMaxBinWin * 2);  // [113] samples sorted by bin
                float2* bsum = srt + kOriSamples + 1;            // [nb]
                for (int i = lane; i < nb; i += 32) cnt[i] = 0;
                __syncwarp();
                float2 val[4];
                int bin[4], pos[4];
                const float fb = (float)nb / kTwoPi;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int j = lane + 32 * r;
                    const bool ok = j < kOriSamples;
                    float rx = 0.f, ry = 0.f;
                    int bb = -1 - lane;  // never matches another lane
                    if (ok) {
                        const float px = x + sigma * c_ori_u[j], py = y + sigma * c_ori_v[j];
                        const float w = c_ori_w[j];
                        const float2 gv = bilinear2(lxy, g.W, g.H, g.P, px, py);  // exact: the window is an argmax
                        rx = w * gv.x;
                        ry = w * gv.y;
                        float ph = atan2f(ry, rx);
                        if (ph < 0.f) ph += kTwoPi;
                        bb = min((int)(ph * fb), nb - 1);
                    }
                    const unsigned peers = __match_any_sync(0xffffffffu, bb);
                    const int base = ok ? cnt[bb] : 0;
                    __syncwarp();
                    const int rank = __popc(peers & ((1u << lane) - 1u));
                    if (ok && rank == 0) cnt[bb] = base + __popc(peers);
                    __syncwarp();
                    val[r] = make_float2(rx, ry);
                    bin[r] = bb;
                    pos[r] = base + rank;
                }
                // exclusive scan of the counts (3 bins per lane, nb <= 96)
                int c3[3], run = 0;
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const int i = 3 * lane + t;
                    c3[t] = i < nb ? cnt[i] : 0;
                    run += c3[t];
                }
                int incl = run;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int tv = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += tv;
                }
                int ex = incl - run;
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const int i = 3 * lane + t;
                    if (i < nb) off[i] = ex;
                    ex += c3[t];
                }
                __syncwarp();
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (lane + 32 * r < kOriSamples) srt[off[bin[r]] + pos[r]] = val[r];
                __syncwarp();
                for (int i = lane; i < nb; i += 32) {
                    float ax = 0.f, ay = 0.f;
                    const int e = off[i] + cnt[i];
                    for (int q = off[i]; q < e; ++q) {
                        ax += srt[q].x;
                        ay += srt[q].y;
                    }
                    bsum[i] = make_float2(ax, ay);
                }
                __syncwarp();
                for (int kw = lane; kw < nwin; kw += 32) {
                    float ax = 0.f, ay = 0.f;
                    int i = 2 * kw - h;
                    if (i < 0) i += nb;
                    for (int q = 0; q < 2 * h; ++q) {
                        const float2 v = bsum[i];
                        ax += v.x;
                        ay += v.y;
                        if (++i == nb) i = 0;
                    }
                    const float m = ax * ax + ay * ay;
                    if (m > best) {
                        best = m;
                        bx = ax;
                        by = ay;
                        bk = kw;
                    }
                }
            } else {  // any other window count: direct scan of the samples for every window
                float4* so = reinterpret_cast<float4*>(sx);  // (phase, w·Lx, w·Ly, -) per sample
#pragma unroll
                for (int j = lane; j < kOriSamples; j += 32) {
                    const float px = x + sigma * c_ori_u[j], py = y + sigma * c_ori_v[j];
                    const float w = c_ori_w[j];
                    const float2 gv = bilinear2(lxy, g.W, g.H, g.P, px, py);
                    const float rx = w * gv.x, ry = w * gv.y;
                    float ph = atan2f(ry, rx);
                    if (ph < 0.f) ph += kTwoPi;
                    so[j] = make_float4(ph, rx, ry, 0.f);
                }
                __syncwarp();
                for (int kw = lane; kw < nwin; kw += 32) {
                    const float th = kTwoPi * (float)kw / (float)nwin;
                    float ax = 0.f, ay = 0.f;
#pragma unroll 4
                    for (int j = 0; j < kOriSamples; ++j) {
                        const float4 e = so[j];  // broadcast read
                        float d = e.x - th;
                        if (d > kPi) d -= kTwoPi;
                        else if (d <= -kPi) d += kTwoPi;
                        const bool in = fabsf(d) < kPi / 6.f;
                        ax += in ? e.y : 0.f;
                        ay += in ? e.z : 0.f;
                    }
                    const float m = ax * ax + ay * ay;
                    if (m > best) {
                        best = m;
                        bx = ax;
                        by = ay;
                        bk = kw;
                    }
                }
            }
            // warp arg-max, ties → lowest window index
            for (int o = 16; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
                const float ox = __shfl_xor_sync(0xffffffffu, bx, o);
                const float oy = __shfl_xor_sync(0xffffffffu, by, o);
                if (ob > best || (ob == best && ok < bk)) {
                    best = ob;
                    bk = ok;
                    bx = ox;
                    by = oy;
                }
            }
            if (best > 0.f) {
                angle = atan2f(by, bx);
                if (angle < 0.f) angle += kTwoPi;
                if (angle >= kTwoPi) angle -= kTwoPi;
            } else {
                angle = 0.f;
                flags = 1;
            }
            __syncwarp();  // done with the orientation buffers
        }
        // ---- M-SURF ----
        float si, co;
        sincosf(angle, &si, &co);
        // lanes walk the rotated axis that runs closest to image x, so a warp's gathers share cache lines
        const bool u_fast = fabsf(co) >= fabsf(si);
#pragma unroll 6
        for (int s = lane; s < 576; s += 32) {
            const int hi = s / 24, lo = s - hi * 24;
            const int p = u_fast ? lo : hi, q = u_fast ? hi : lo;
            const float u = (float)p - 11.5f, v = (float)q - 11.5f;
            const float px = x + sigma * (u * co - v * si);
            const float py = y + sigma * (u * si + v * co);
            // hardware bilinear filtering (texel centres at +0.5; clamped addressing = clamped taps, A14/A16)
            const float2 gv = tex2D<float2>(tex, px + 0.5f, py + 0.5f);
            const float gx = gv.x, gy = gv.y;
            sx[p * kSP + q] = gx * co + gy * si;  // pitch 25: conflict-free for lanes along p or q
            sy[p * kSP + q] = -gx * si + gy * co;
        }
        __syncwarp();
        const int sr = lane >> 1, half = lane & 1;
        const int a = sr & 3, b = sr >> 2;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        for (int i = half; i < 9; i += 2) {
            const int p = 5 * a + i;
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const int q = 5 * b + j;
                const float w = c_w1[i * 9 + j];
                const float du = w * sx[p * kSP + q], dv = w * sy[p * kSP + q];
                s0 += du;
                s1 += dv;
                s2 += fabsf(du);
                s3 += fabsf(dv);
            }
        }
        s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        s3 += __shfl_xor_sync(0xffffffffu, s3, 1);
        const float w2 = c_w2[sr];
        s0 *= w2;
        s1 *= w2;
        s2 *= w2;
        s3 *= w2;
        float n2 = half == 0 ? s0 * s0 + s1 * s1 + s2 * s2 + s3 * s3 : 0.f;
        for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        const float inv = n2 > 0.f ? rsqrtf(n2) : 0.f;
        if (half == 0) {
            float4 out = make_float4(s0 * inv, s1 * inv, s2 * inv, s3 * inv);
            reinterpret_cast<float4*>(desc + ((size_t)img * cap + k) * 64)[sr] = out;
        }
        if (lane == 0 && !keep_angle) {
            kp->angle = angle;
            kp->flags = flags;
        }
        __syncwarp();
    }
}

}  // namespace

void init_describe_tables() {
    float u[kOriSamples], v[kOriSamples], w[kOriSamples];
    int n = 0;
    for (int vv = -6; vv <= 6; ++vv)
        for (int uu = -6; uu <= 6; ++uu) {
            if (uu * uu + vv * vv > 36) continue;
            u[n] = (float)uu;
            v[n] = (float)vv;
            w[n] = (float)exp(-(double)(uu * uu + vv * vv) / 12.5);
            ++n;
        }
    float w1[81], w2[16];
    for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) w1[i * 9 + j] = (float)exp(-(double)((i - 4) * (i - 4) + (j - 4) * (j - 4)) / 12.5);
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) w2[4 * b + a] = (float)exp(-((a - 1.5) * (a - 1.5) + (b - 1.5) * (b - 1.5)) / 4.5);
    cudaMemcpyToSymbol(c_ori_u, u, sizeof(u));
    cudaMemcpyToSymbol(c_ori_v, v, sizeof(v));
    cudaMemcpyToSymbol(c_ori_w, w, sizeof(w));
    cudaMemcpyToSymbol(c_w1, w1, sizeof(w1));
    cudaMemcpyToSymbol(c_w2, w2, sizeof(w2));
}

void launch_describe(const float2* Lxy, const cudaTextureObject_t* texs, size_t img_stride, Geom g, int nimg, int N,
                     kaze_keypoint* kps, const int* counts, int cap, float* desc, int nwin, int keep_angle,
                     cudaStream_t s) {
    // Persistent grid of exactly one wave: the CTAs that fit on every SM at once (registers limit it to 4 of 256
    // threads).  A grid larger than one wave leaves the surplus CTAs' share of the static keypoint stride to a
    // second, mostly idle wave (measured: 148·5 CTAs = 1.25 waves).
    static int grid = 0;
    if (grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_describe, 256, 0);
        grid = sms * (per_sm > 0 ? per_sm : 1);
    }
    k_describe<<<grid, 256, 0, s>>>(Lxy, texs, img_stride, g, nimg, kps, counts, cap, desc, nwin, keep_angle, N);
}

}  // namespace kz
