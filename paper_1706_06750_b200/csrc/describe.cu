// describe.cu — dominant orientation (A14) and 64-D M-SURF (A15).
//
// One warp per keypoint over the FLAT list of all keypoints of all levels and images (the paper's load-balancing
// remedy: "all the image scales are computed at the same time"), persistent grid of one full wave (occupancy-sized).
//   orientation: 113 samples at kp + σ(u, v), u² + v² <= 36, spread over the lanes; Gaussian weight
//                exp(−(u²+v²)/12.5) (std 2.5σ); the weighted (Lx, Ly) vectors go to shared memory; lanes own the
//                window centres θ_k = 2πk/nwin and sum the vectors within ±π/6; a warp arg-max (first k on
//                ties) picks the longest sum; angle = atan2 of it in [0, 2π).
//   M-SURF:      24 x 24 samples at step σ rotated by the angle, bilinear (Lx, Ly) rotated into the keypoint
//                frame (du, dv); lane t < 24 walks grid line t in registers and keeps, per subregion along the walk,
//                the line sums weighted by the separable Gaussian (std 2.5 about the subregion centre); a cross-line
//                pass over shared memory sums 9 lines per subregion, the 4x4 mask (std 1.5) weights it, the warp
//                normalises the 64-vector and writes it with coalesced stores.  (Measured on B200: staging all 576
//                samples in shared memory and summing 9 x 9 windows per lane pair cost 2-way bank conflicts on
//                every access — 47% of the kernel's shared wavefronts — and 26.4 ms per 256-image step.)
#include "kaze_internal.cuh"

namespace kz {

namespace {

constexpr int kOriSamples = 113;
__constant__ float c_ori_u[kOriSamples], c_ori_v[kOriSamples], c_ori_w[kOriSamples];
__constant__ float c_g1[9];   // exp(-(i-4)^2 / (2 * 2.5^2)), i = 0..8: w1(i, j) = g1(i)·g1(j) (separable, A15)
__constant__ float c_w2[16];  // exp(-((a-1.5)^2 + (b-1.5)^2) / (2 * 1.5^2)), index 4b + a

constexpr float kTwoPi = 6.283185307179586f;
constexpr float kPi = 3.141592653589793f;

// atan2 for the orientation BIN of a sample (|error| <= 1.1e-7 rad, like atan2f's 2 ulp; the final angle keeps
// atan2f): octant reduction, a = min/max in [0, 1], atan(a) = a + a·s·p(s), s = a², p of degree 6 fitted to
// minimise the max fp32 error on [0, 1]; about half of atan2f's instructions.
__device__ __forceinline__ float atan2_bin(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(mx));
    const float a = mx > 0.f ? mn * r : 0.f;
    const float q = a * a;
    float p = -0.004355322103947401f;
    p = fmaf(p, q, 0.023039856925606728f);
    p = fmaf(p, q, -0.057773225009441376f);
    p = fmaf(p, q, 0.09794210642576218f);
    p = fmaf(p, q, -0.13976573944091797f);
    p = fmaf(p, q, 0.19962702691555023f);
    p = fmaf(p, q, -0.3333165943622589f);
    float t = fmaf(a * q, p, a);
    if (ay > ax) t = 1.5707963267948966f - t;
    if (x < 0.f) t = 3.141592653589793f - t;
    return y < 0.f ? -t : t;
}

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
constexpr int kLP = 17;         // pitch of the staged per-line subregion sums (24 lines x 16)
constexpr int kWarpBuf = 640;   // floats of shared scratch per warp (orientation sort: 612)
constexpr int kMaxBinWin = 48;  // binned orientation path: nwin % 6 == 0 and nwin <= 48 (2·nwin <= 96 bins)

// Five CTAs per SM (48 registers): 23.4 ms per 256-image step vs 24.9 at four (59 registers) and 24.2 at six.
__global__ void __launch_bounds__(256, 5) k_describe(const float2* __restrict__ Lxy,
                                                  const cudaTextureObject_t* __restrict__ texs, size_t img_stride, Geom g, int nimg, kaze_keypoint* __restrict__ kps,
                                                  const int* __restrict__ counts, int cap, float* __restrict__ desc,
                                                  int nwin, int keep_angle, int N, int lvl_lo, int lvl_hi,
                                                  int* __restrict__ work) {
    KZ_PDL_PROLOGUE();
    __shared__ int pre[kMaxBatch + 1];
    __shared__ __align__(16) float sbuf[kWarps][kWarpBuf];
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
    // CTA b's warps take 8 consecutive keypoints, then jump by the grid: the whole grid works on one narrow window
    // of the (image, level, y, x)-ordered list, so the planes it samples stay in L2.  (A contiguous range per CTA —
    // more L1 sharing, but the grid spread over every image and level at once — measured 48.8 vs 24.7 ms; 2 or 4
    // consecutive keypoints per warp per round 24.2 / 27.8 vs 23.5.)
    int img = 0;  // f only grows, so the image search resumes where the previous keypoint left it
    // Work distribution: with `work` (a zeroed device counter) each warp takes the next keypoint of the flat
    // (image, level, y, x) list when it is free, so the grid still sweeps one narrow window of the list (planes
    // stay L2-resident) and no warp idles while another finishes a static share; without it, a static stride.
    const int stride = gridDim.x * kWarps;
    auto next = [&](int cur) {
        if (!work) return cur < 0 ? (int)(blockIdx.x * kWarps + warp) : cur + stride;
        int v = 0;
        if (lane == 0) v = atomicAdd(work, 1);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    for (int f = next(-1); f < total; f = next(f)) {
        while (img + 1 < nimg && pre[img + 1] <= f) ++img;
        const int k = f - pre[img];
        kaze_keypoint* kp = kps + (size_t)img * cap + k;
        const float x = kp->x, y = kp->y, sigma = kp->sigma;
        const int level = kp->level;
        if (level < lvl_lo || level > lvl_hi) {  // warp-uniform: no sampleable (Lx, Ly) planes at this level
            float* dk = desc + ((size_t)img * cap + k) * 64;
            dk[lane] = 0.f;
            dk[lane + 32] = 0.f;
            if (lane == 0) {
                if (!keep_angle) kp->angle = 0.f;
                kp->flags = 1;
            }
            __syncwarp();
            continue;
        }
        const float2* lxy = Lxy + img * img_stride + (size_t)level * g.plane;
        // The texture handle is the same for the whole warp; broadcasting it from lane 0 lets ptxas prove that, so
        // every tex2D below takes the handle from a uniform register directly.  (Loaded per lane, the handle is
        // "maybe divergent" to the compiler, which then wraps each fetch in a uniformisation loop — R2UR + BRA.U.ANY
        // — and issues the 24 fetches of a grid line one at a time, each waiting out the full fetch latency.)
        cudaTextureObject_t tex = texs[img * N + level];
        {
            const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)tex, 0);
            const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)(tex >> 32), 0);
            tex = ((cudaTextureObject_t)hi << 32) | lo;
        }
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
                        float ph = atan2_bin(ry, rx);
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
                // Window k = bins [2k − h, 2k + h): h whole bin pairs starting at bins of parity o = h & 1, so the
                // window sums pair sums Q_j = bin[2j + o] + bin[2j + o + 1], j = k − (h + o)/2 .. + h − 1 (mod nwin):
                // h adds per window instead of 2h (srt is free again and holds Q).
                float2* qs = srt;
                const int o = h & 1;
                for (int j = lane; j < nwin; j += 32) {
                    const float2 a = bsum[2 * j + o], b = bsum[(2 * j + o + 1) % nb];
                    qs[j] = make_float2(a.x + b.x, a.y + b.y);
                }
                __syncwarp();
                for (int kw = lane; kw < nwin; kw += 32) {
                    float ax = 0.f, ay = 0.f;
                    int i = kw - (h + o) / 2;
                    if (i < 0) i += nwin;
                    for (int q = 0; q < h; ++q) {
                        const float2 v = qs[i];
                        ax += v.x;
                        ay += v.y;
                        if (++i == nwin) i = 0;
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
        // Grid sample (p, q) sits at u = p − 11.5, v = q − 11.5 (steps of σ, keypoint frame).  Lane t < 24 owns one
        // grid line across the rotated axis that runs closest to image x (lanes along u when |cos| >= |sin|), so the
        // warp's 24 gathers of a step lie on one line and share cache lines; it walks the line's 24 samples and, as
        // the subregion weight is separable (w1(i, j) = g(i)·g(j), g(i) = exp(−(i−4)²/12.5)), accumulates g-weighted
        // line sums of the four subregions along the walk.  The cross-line pass then sums 9 lines per subregion.
        const bool u_fast = fabsf(co) >= fabsf(si);
        float acc[4][4];  // [subregion along the walk][Σdu, Σdv, Σ|du|, Σ|dv|]
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) acc[r][q4] = 0.f;
        if (lane < 24) {
#pragma unroll
            for (int t = 0; t < 24; ++t) {
                const int p = u_fast ? lane : t, q = u_fast ? t : lane;
                const float u = (float)p - 11.5f, v = (float)q - 11.5f;
                const float px = x + sigma * (u * co - v * si);
                const float py = y + sigma * (u * si + v * co);
                // hardware bilinear filtering (texel centres at +0.5; clamped addressing = clamped taps, A14/A16)
                const float2 gv = tex2D<float2>(tex, px + 0.5f, py + 0.5f);
                const float du = gv.x * co + gv.y * si, dv = -gv.x * si + gv.y * co;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = t - 5 * r;  // compile-time: sample t is row i of subregion r iff 0 <= i <= 8
                    if (i < 0 || i > 8) continue;
                    const float wg = c_g1[i];
                    acc[r][0] = fmaf(wg, du, acc[r][0]);
                    acc[r][1] = fmaf(wg, dv, acc[r][1]);
                    acc[r][2] = fmaf(wg, fabsf(du), acc[r][2]);
                    acc[r][3] = fmaf(wg, fabsf(dv), acc[r][3]);
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) sx[lane * kLP + 4 * r + q4] = acc[r][q4];
        }
        __syncwarp();
        // output o = 4(4b + a) + j (A15): lane L computes o = L and o = L + 32
        float ov[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int o = lane + 32 * h, sr = o >> 2, j = o & 3, a = sr & 3, b = sr >> 2;
            const int l = u_fast ? a : b, r = u_fast ? b : a;  // subregion index across lines / along the walk
            float sum = 0.f;
#pragma unroll
            for (int i = 0; i < 9; ++i) sum = fmaf(c_g1[i], sx[(5 * l + i) * kLP + 4 * r + j], sum);
            ov[h] = sum * c_w2[sr];
        }
        float n2 = ov[0] * ov[0] + ov[1] * ov[1];
        for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        const float inv = n2 > 0.f ? rsqrtf(n2) : 0.f;
        float* dk = desc + ((size_t)img * cap + k) * 64;
        dk[lane] = ov[0] * inv;
        dk[lane + 32] = ov[1] * inv;
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
    float g1[9], w2[16];
    for (int i = 0; i < 9; ++i) g1[i] = (float)exp(-(double)((i - 4) * (i - 4)) / 12.5);
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) w2[4 * b + a] = (float)exp(-((a - 1.5) * (a - 1.5) + (b - 1.5) * (b - 1.5)) / 4.5);
    cudaMemcpyToSymbol(c_ori_u, u, sizeof(u));
    cudaMemcpyToSymbol(c_ori_v, v, sizeof(v));
    cudaMemcpyToSymbol(c_ori_w, w, sizeof(w));
    cudaMemcpyToSymbol(c_g1, g1, sizeof(g1));
    cudaMemcpyToSymbol(c_w2, w2, sizeof(w2));
}

void launch_describe(const float2* Lxy, const cudaTextureObject_t* texs, size_t img_stride, Geom g, int nimg, int N,
                     int lvl_lo, int lvl_hi, int* work, int overlapped, kaze_keypoint* kps, const int* counts, int cap, float* desc, int nwin, int keep_angle,
                     cudaStream_t s) {
    // Persistent grid of exactly one wave: the CTAs that fit on every SM at once (registers limit it to 4 of 256
    // threads).  A grid larger than one wave leaves the surplus CTAs' share of the static keypoint stride to a
    // second, mostly idle wave (measured: 148·5 CTAs = 1.25 waves).
    int per_sm = 0;  // (a per-device figure: cheap, and correct when contexts on other devices share the process)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_describe, 256, 0);
    // Overlapped with the next chunk's scale space, a smaller persistent grid (3 CTAs per SM) leaves the SMs room for
    // those passes' CTAs (256-image step, 32 per launch: 149.0 vs 149.6 ms at the full 5); KAZE_DESC_OCC overrides.
    static const int occ = tune_knob("KAZE_DESC_OCC", 3);
    if (overlapped && occ > 0 && per_sm > occ) per_sm = occ;
    const int grid = device_sm_count() * (per_sm > 0 ? per_sm : 1);
    kz_launch(k_describe, dim3(grid), dim3(256), 0, s, Lxy, texs, img_stride, g, nimg, kps, counts, cap, desc, nwin, keep_angle, N, lvl_lo, lvl_hi, work);
}

}  // namespace kz
