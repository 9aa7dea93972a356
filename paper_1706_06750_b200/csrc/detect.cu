// detect.cu — 3x3x3 extrema, edge test, 2-D sub-pixel fit and deterministic compaction (sm_100a).
//
// P:L207-214 and P:L263-281, readings A11-A13: a pixel (x, y) of level i in 1..N−2, at least one pixel from the
// border, is a keypoint iff Ldet > threshold, Ldet is strictly greater than its 26 neighbours in levels i−1, i,
// i+1, the Hessian of the response surface passes Det > 0 and Tr²/Det < (r+1)²/r (Eq. 12; Tr = Dxx + Dyy), and
// the quadratic fit offset δ = −H⁻¹∇D has |δx|, |δy| <= 1.
//
// Compaction is deterministic and ordered by (level, y, x) without a sort:
//   nms_mark : warps streaming 32-column strips down the rows — ballots produce a 1-bit-per-pixel candidate bitmap;
//              k_rowcount turns it into per-row candidate counts;
//   kp_scan  : one CTA per image — exclusive scan of the row counts → row offsets, total → d_counts;
//   kp_emit  : one warp per (image, level, row) — rank of each set bit = row offset + popcounts before it; the
//              sub-pixel fit is re-evaluated (same fp32 code as the mark pass, so the same decision) and the
//              32-byte keypoint is written if its rank is below the capacity.
#include "kaze_internal.cuh"

namespace kz {

namespace {

// Edge test + sub-pixel fit on the 3x3 patch D[r][c] (r = dy+1, c = dx+1).  Returns keep.
__device__ __forceinline__ bool refine(const float (&D)[3][3], float edge_ratio, float& ox, float& oy) {
    const float cv = D[1][1];
    const float dxx = D[1][2] + D[1][0] - 2.f * cv;
    const float dyy = D[2][1] + D[0][1] - 2.f * cv;
    const float dxy = 0.25f * (D[2][2] + D[0][0] - D[0][2] - D[2][0]);
    const float gx = 0.5f * (D[1][2] - D[1][0]);
    const float gy = 0.5f * (D[2][1] - D[0][1]);
    const float det = dxx * dyy - dxy * dxy;
    if (edge_ratio > 0.f) {
        const float tr = dxx + dyy;
        if (!(det > 0.f)) return false;
        if (!(tr * tr / det < (edge_ratio + 1.f) * (edge_ratio + 1.f) / edge_ratio)) return false;
    }
    if (fabsf(det) < 1e-12f) return false;
    ox = -(dyy * gx - dxy * gy) / det;
    oy = -(dxx * gy - dxy * gx) / det;
    return fabsf(ox) <= 1.f && fabsf(oy) <= 1.f;
}

__device__ __forceinline__ bool is_keypoint(const float* __restrict__ Dm, const float* __restrict__ D0,
                                            const float* __restrict__ Dp, int P, int x, int y, float thr, float er,
                                            float& ox, float& oy, float& v) {
    const size_t o = (size_t)y * P + x;
    v = __ldg(D0 + o);
    if (!(v > thr)) return false;
    float patch[3][3];
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const size_t q = o + (ptrdiff_t)dy * P + dx;
            float a = __ldg(Dm + q), c = __ldg(Dp + q);
            if (!(v > a) || !(v > c)) return false;
            if (dx != 0 || dy != 0) {
                float b = __ldg(D0 + q);
                if (!(v > b)) return false;
                patch[dy + 1][dx + 1] = b;
            }
        }
    patch[1][1] = v;
    return refine(patch, er, ox, oy);
}

// nms_mark: one WARP per (32-column strip, NSEG-row segment, level, image), streaming down the rows.  Lane l owns
// column x0+l and keeps, for each of the levels i-1, i, i+1, the last three rows of its column in registers (lanes 0
// and 31 also keep the halo columns x0-1 / x0+32).  The 26-neighbour maximum is
//   max(vmax_{i-1}, vmax_{i+1} over columns x-1..x+1;  vmax_i over x-1, x+1;  D_i(x, y±1))
// with vmax = vertical 3-maximum, the column neighbours coming from shuffles: ~30 instructions per pixel, 3
// coalesced loads per pixel, no shared memory, no barriers.  Only candidates run the edge test / sub-pixel fit.
// The warp writes the row's 32-bit candidate word; row counts come from k_rowcount.
constexpr int NSEG = 64;

__global__ void __launch_bounds__(256) k_nms_mark(const float* __restrict__ Ldet, size_t img_stride, Geom g, int N,
                                                  DetectParams dp, uint32_t* __restrict__ bitmap) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int words = (g.W + 31) / 32;
    if (strip >= words) return;  // warp-uniform
    const int x0 = strip * 32, x = x0 + lane;
    const int y0 = blockIdx.y * NSEG;
    const int li = blockIdx.z % (N - 2), img = blockIdx.z / (N - 2), level = li + 1;
    const int W = g.W, H = g.H;
    const float* D1 = Ldet + img * img_stride + (size_t)level * g.plane;
    const float* D0 = D1 - g.plane;
    const float* D2 = D1 + g.plane;
    const int xc = min(x, W - 1);
    const bool halo = lane == 0 || lane == 31;
    const int xh = lane == 0 ? max(x0 - 1, 0) : min(x0 + 32, W - 1);
    // windows: [0] = row y-1, [1] = y, [2] = y+1 (own column), h* = halo column
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
    float ha0 = 0.f, ha1 = 0.f, ha2 = 0.f, hb0 = 0.f, hb1 = 0.f, hb2 = 0.f, hc0 = 0.f, hc1 = 0.f, hc2 = 0.f;
    const int ylast = min(y0 + NSEG, H - 1);  // last row loaded (the row below the last output row)
    uint32_t* bm = bitmap + (((size_t)img * (N - 2) + li) * H) * words + strip;
    // software pipeline: the next row's loads are issued before the current row is consumed
    size_t ro = (size_t)max(y0 - 1, 0) * g.P;
    float na = __ldg(D0 + ro + xc), nb = __ldg(D1 + ro + xc), nc = __ldg(D2 + ro + xc);
    float nha = 0.f, nhb = 0.f, nhc = 0.f;
    if (halo) {
        nha = __ldg(D0 + ro + xh);
        nhb = __ldg(D1 + ro + xh);
        nhc = __ldg(D2 + ro + xh);
    }
    for (int r = y0 - 1; r <= ylast; ++r) {
        a0 = a1; a1 = a2; a2 = na;
        b0 = b1; b1 = b2; b2 = nb;
        c0 = c1; c1 = c2; c2 = nc;
        if (halo) {
            ha0 = ha1; ha1 = ha2; ha2 = nha;
            hb0 = hb1; hb1 = hb2; hb2 = nhb;
            hc0 = hc1; hc1 = hc2; hc2 = nhc;
        }
        if (r < ylast) {
            ro = (size_t)(r + 1) * g.P;
            na = __ldg(D0 + ro + xc);
            nb = __ldg(D1 + ro + xc);
            nc = __ldg(D2 + ro + xc);
            if (halo) {
                nha = __ldg(D0 + ro + xh);
                nhb = __ldg(D1 + ro + xh);
                nhc = __ldg(D2 + ro + xh);
            }
        }
        const int y = r - 1;  // the window now holds rows y-1, y, y+1
        if (y < y0) continue;
        const float va = fmaxf(a0, fmaxf(a1, a2)), vc = fmaxf(c0, fmaxf(c1, c2)), vb = fmaxf(b0, fmaxf(b1, b2));
        float val = __shfl_up_sync(0xffffffffu, va, 1), var = __shfl_down_sync(0xffffffffu, va, 1);
        float vcl = __shfl_up_sync(0xffffffffu, vc, 1), vcr = __shfl_down_sync(0xffffffffu, vc, 1);
        float vbl = __shfl_up_sync(0xffffffffu, vb, 1), vbr = __shfl_down_sync(0xffffffffu, vb, 1);
        if (halo) {
            const float hva = fmaxf(ha0, fmaxf(ha1, ha2)), hvc = fmaxf(hc0, fmaxf(hc1, hc2));
            const float hvb = fmaxf(hb0, fmaxf(hb1, hb2));
            if (lane == 0) { val = hva; vcl = hvc; vbl = hvb; }
            else { var = hva; vcr = hvc; vbr = hvb; }
        }
        float m = fmaxf(fmaxf(val, va), fmaxf(var, vc));
        m = fmaxf(m, fmaxf(fmaxf(vcl, vcr), fmaxf(vbl, vbr)));
        m = fmaxf(m, fmaxf(b0, b2));
        bool k = (x >= 1 && x <= W - 2 && y >= 1 && y <= H - 2) && b1 > dp.threshold && b1 > m;
        if (__any_sync(0xffffffffu, k)) {  // rare: gather the level-i 3x3 patch and fit
            float l0 = __shfl_up_sync(0xffffffffu, b0, 1), l1 = __shfl_up_sync(0xffffffffu, b1, 1);
            float l2 = __shfl_up_sync(0xffffffffu, b2, 1);
            float q0 = __shfl_down_sync(0xffffffffu, b0, 1), q1 = __shfl_down_sync(0xffffffffu, b1, 1);
            float q2 = __shfl_down_sync(0xffffffffu, b2, 1);
            if (lane == 0) { l0 = hb0; l1 = hb1; l2 = hb2; }
            if (lane == 31) { q0 = hb0; q1 = hb1; q2 = hb2; }
            if (k) {
                const float patch[3][3] = {{l0, b0, q0}, {l1, b1, q1}, {l2, b2, q2}};
                float ox, oy;
                k = refine(patch, dp.edge_ratio, ox, oy);
            }
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, k);
        if (lane == 0 && y < H) bm[(size_t)y * words] = bits;
    }
    // the last image row is never a window centre above; it has no candidates (border)
    if (lane == 0 && y0 + NSEG >= H && H - 1 >= y0) bm[(size_t)(H - 1) * words] = 0u;
}

// Row candidate counts from the bitmap: one warp per (image, level, row).
__global__ void __launch_bounds__(256) k_rowcount(const uint32_t* __restrict__ bitmap, int words, int total_rows,
                                                  int* __restrict__ rowcnt) {
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= total_rows) return;
    const uint32_t* bm = bitmap + (size_t)q * words;
    int c = 0;
    for (int w = lane; w < words; w += 32) c += __popc(bm[w]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) rowcnt[q] = c;
}

// One CTA per image: exclusive scan of R row counts.
__global__ void __launch_bounds__(1024) k_kp_scan(const int* __restrict__ rowcnt, int R, int* __restrict__ rowoff,
                                                  int* __restrict__ counts) {
    __shared__ int wsum[32];
    const int img = blockIdx.x;
    const int* rc = rowcnt + (size_t)img * R;
    int* ro = rowoff + (size_t)img * R;
    const int per = (R + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(b + per, R);
    int local = 0;
    for (int i = b; i < e; ++i) local += rc[i];
    // block exclusive scan of `local`
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        wsum[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    int run = incl - local + (warp > 0 ? wsum[warp - 1] : 0);
    for (int i = b; i < e; ++i) {
        ro[i] = run;
        run += rc[i];
    }
    if (threadIdx.x == blockDim.x - 1) counts[img] = run;
}

// One WARP per (image, level, row); 8 rows per CTA.  Lane w of a 32-word step owns bitmap word w: an inclusive warp
// scan of the word popcounts gives each word's rank base, and the lane walks its set bits in x order.
__global__ void __launch_bounds__(256) k_kp_emit(const float* __restrict__ Ldet, size_t img_stride, Geom g,
                                                 LevelTable lt, DetectParams dp, const uint32_t* __restrict__ bitmap,
                                                 const int* __restrict__ rowcnt, const int* __restrict__ rowoff,
                                                 kaze_keypoint* __restrict__ kps, int total_rows) {
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5);  // flat row id over (img, level-1, y)
    if (q >= total_rows) return;
    if (rowcnt[q] == 0) return;  // warp-uniform
    const int N = lt.n;
    const int y = q % g.H, rest = q / g.H, li = rest % (N - 2), img = rest / (N - 2), level = li + 1;
    const int words = (g.W + 31) / 32;
    const uint32_t* bm = bitmap + (size_t)q * words;
    const float* D0 = Ldet + img * img_stride + (size_t)level * g.plane;
    int run = rowoff[q];
    for (int w0 = 0; w0 < words; w0 += 32) {
        uint32_t word = (w0 + lane < words) ? bm[w0 + lane] : 0u;
        const int c = __popc(word);
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        int rank = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
        while (word) {
            const int bit = __ffs(word) - 1;
            word &= word - 1;
            if (rank < dp.cap) {
                const int x = (w0 + lane) * 32 + bit;
                float ox = 0.f, oy = 0.f, v = 0.f;
                is_keypoint(D0 - g.plane, D0, D0 + g.plane, g.P, x, y, dp.threshold, dp.edge_ratio, ox, oy, v);
                kaze_keypoint kp;
                kp.x = (float)x + ox;
                kp.y = (float)y + oy;
                kp.sigma = lt.sigma[level];
                kp.response = v;
                kp.angle = 0.f;
                kp.level = level;
                kp.octave = (int16_t)(level / lt.S);
                kp.sublevel = (int16_t)(level % lt.S);
                kp.flags = 0;
                kps[(size_t)img * dp.cap + rank] = kp;
            }
            ++rank;
        }
    }
}

}  // namespace

void launch_nms_mark(const float* Ldet, size_t img_stride, Geom g, int nimg, int N, DetectParams dp, uint32_t* bitmap,
                     int* rowcnt, cudaStream_t s) {
    const int words = (g.W + 31) / 32;
    dim3 grid((words + 7) / 8, (g.H + NSEG - 1) / NSEG, nimg * (N - 2));
    k_nms_mark<<<grid, 256, 0, s>>>(Ldet, img_stride, g, N, dp, bitmap);
    const int total = g.H * (N - 2) * nimg;
    k_rowcount<<<(total + 7) / 8, 256, 0, s>>>(bitmap, words, total, rowcnt);
}

void launch_kp_scan(const int* rowcnt, int rows_per_img, int nimg, int* rowoff, int* counts, cudaStream_t s) {
    k_kp_scan<<<nimg, 1024, 0, s>>>(rowcnt, rows_per_img, rowoff, counts);
}

void launch_kp_emit(const float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt, DetectParams dp,
                    const uint32_t* bitmap, const int* rowcnt, const int* rowoff, kaze_keypoint* kps, cudaStream_t s) {
    const int total = g.H * (lt.n - 2) * nimg;
    k_kp_emit<<<(total + 7) / 8, 256, 0, s>>>(Ldet, img_stride, g, lt, dp, bitmap, rowcnt, rowoff, kps, total);
}

}  // namespace kz
