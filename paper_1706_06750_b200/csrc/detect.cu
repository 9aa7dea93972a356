// detect.cu — 3x3x3 extrema, edge test, 2-D sub-pixel fit and deterministic compaction (sm_100a).
//
// P:L207-214 and P:L263-281, readings A11-A13: a pixel (x, y) of level i in 1..N−2, at least one pixel from the
// border, is a keypoint iff Ldet > threshold, Ldet is strictly greater than its 26 neighbours in levels i−1, i,
// i+1, the Hessian of the response surface passes Det > 0 and Tr²/Det < (r+1)²/r (Eq. 12; Tr = Dxx + Dyy), and
// the quadratic fit offset δ = −H⁻¹∇D has |δx|, |δy| <= 1.
//
// Compaction is deterministic and ordered by (level, y, x) without a sort:
//   nms_mark : one CTA per (image, level, row) — warp ballots produce a 1-bit-per-pixel candidate bitmap and the
//              row's candidate count;
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

// nms_mark tile: 256 columns x NY rows of one level of one image, one thread per column.  Each thread loads its
// column of the three levels (NY+2 rows each) into registers with coalesced row loads, forms the vertical 3-maxima
// in registers and publishes them in shared memory; the 26-neighbour maximum of a pixel is then
//   max( V_{i-1}[c-1..c+1][r], V_{i+1}[c-1..c+1][r], V_i[c±1][r], D_i[c][r±1] )
// (V = vertical 3-max), a handful of operations per pixel.  Only candidates run the edge test / sub-pixel fit.
constexpr int NX = 256, NY = 8;

__global__ void __launch_bounds__(256) k_nms_mark(const float* __restrict__ Ldet, size_t img_stride, Geom g, int N,
                                                  DetectParams dp, uint32_t* __restrict__ bitmap,
                                                  int* __restrict__ rowcnt) {
    __shared__ float V[3][NY][NX + 2];   // vertical 3-max per level, row r (output rows), column c (tile coords)
    __shared__ float C1[NY + 2][NX + 2]; // level-i values (for the 3x3 patch of candidates)
    __shared__ int rc[NY];
    const int x0 = blockIdx.x * NX, y0 = blockIdx.y * NY;
    const int li = blockIdx.z % (N - 2), img = blockIdx.z / (N - 2), level = li + 1;
    const float* D0 = Ldet + img * img_stride + (size_t)level * g.plane;
    const int tid = threadIdx.x;
    if (tid < NY) rc[tid] = 0;
    // columns handled by this thread: its own (tile column tid+1) and, for threads 0 / 1, the halo columns 0 / NX+1
    for (int pass = 0; pass < 2; ++pass) {
        int col;
        if (pass == 0) col = tid + 1;
        else if (tid == 0) col = 0;
        else if (tid == 1) col = NX + 1;
        else break;
        const int gx = clampi(x0 - 1 + col, 0, g.W - 1);
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            const float* Dl = D0 + (ptrdiff_t)(l - 1) * (ptrdiff_t)g.plane + gx;
            float v[NY + 2];
#pragma unroll
            for (int r = 0; r < NY + 2; ++r) v[r] = __ldg(Dl + (size_t)clampi(y0 - 1 + r, 0, g.H - 1) * g.P);
#pragma unroll
            for (int r = 0; r < NY; ++r) V[l][r][col] = fmaxf(v[r], fmaxf(v[r + 1], v[r + 2]));
            if (l == 1) {
#pragma unroll
                for (int r = 0; r < NY + 2; ++r) C1[r][col] = v[r];
            }
        }
    }
    __syncthreads();
    const int words = (g.W + 31) / 32;
    const int lane = tid & 31, warp = tid >> 5;
    const int x = x0 + tid, c = tid + 1;
#pragma unroll 1
    for (int r = 0; r < NY; ++r) {
        const int y = y0 + r;
        bool k = false;
        if (y >= 1 && y <= g.H - 2 && x >= 1 && x <= g.W - 2) {
            const float v = C1[r + 1][c];
            float m = fmaxf(fmaxf(V[0][r][c - 1], V[0][r][c]), V[0][r][c + 1]);
            m = fmaxf(m, fmaxf(fmaxf(V[2][r][c - 1], V[2][r][c]), V[2][r][c + 1]));
            m = fmaxf(m, fmaxf(V[1][r][c - 1], V[1][r][c + 1]));
            m = fmaxf(m, fmaxf(C1[r][c], C1[r + 2][c]));
            if (v > dp.threshold && v > m) {
                float patch[3][3];
#pragma unroll
                for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) patch[dy][dx] = C1[r + dy][c - 1 + dx];
                float ox, oy;
                k = refine(patch, dp.edge_ratio, ox, oy);
            }
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, k);
        if (lane == 0 && y < g.H && x0 + warp * 32 < g.W) {
            const size_t row = ((size_t)img * (N - 2) + li) * g.H + y;
            bitmap[row * words + (x0 >> 5) + warp] = bits;
            if (bits) atomicAdd(&rc[r], __popc(bits));
        }
    }
    __syncthreads();
    if (tid < NY && y0 + tid < g.H && rc[tid]) atomicAdd(&rowcnt[((size_t)img * (N - 2) + li) * g.H + y0 + tid], rc[tid]);
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
    cudaMemsetAsync(rowcnt, 0, sizeof(int) * (size_t)nimg * (N - 2) * g.H, s);
    dim3 grid((g.W + NX - 1) / NX, (g.H + NY - 1) / NY, nimg * (N - 2));
    k_nms_mark<<<grid, 256, 0, s>>>(Ldet, img_stride, g, N, dp, bitmap, rowcnt);
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
