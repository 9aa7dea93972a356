// kaze_api.cu — the C ABI of include/kaze.h: context, arena, level schedule, orchestration of the sm_100a
// kernels on the caller's stream, CUDA-graph capture/replay of whole chunks (run_chunk), the pipelined
// host-buffer path, per-kernel event profiling, and the host side of programmatic dependent launch.
//
// Host-side arithmetic kept here (schedule, Gaussian taps, τ_i) is this product's own; it shares nothing with
// oracle/ (DESIGN.md §2).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "kaze_internal.cuh"

using namespace kz;

namespace {

enum KernelClass {
    KC_PREFILTER = 0,
    KC_GRAD_L1,
    KC_KHIST,
    KC_KFINAL,
    KC_COND,
    KC_AOS_COLS,
    KC_AOS_ROWS,
    KC_HESSIAN,
    KC_NMS_MARK,
    KC_KP_SCAN,
    KC_KP_EMIT,
    KC_DESCRIBE,
    KC_FED,
    KC_COUNT
};
const char* kKernelNames[KC_COUNT] = {"prefilter", "grad_l1",  "k_hist",   "k_final",
                                      "cond",      "aos_cols", "aos_rows", "hessian",
                                      "nms_mark",  "kp_scan",  "kp_emit",  "describe", "fed"};

struct ProfRec {
    int kc;
    cudaEvent_t e0, e1;
    double bytes;
    int nk;
};

}  // namespace

struct kaze_ctx {
    kaze_params p;
    int device = 0;
    int N = 0;
    // schedule (host, double; A3/A9)
    double sigma[kMaxLevels], t[kMaxLevels];
    int step[kMaxLevels];
    GaussTaps g0{}, g1{};
    LevelTable lt{};
    std::vector<std::vector<float>> fed;  // scheme FED: level i's cycle step sizes in execution order (A20, A21)
    // arena
    int Pmax = 0;
    size_t plane_max = 0;
    float *Lt = nullptr, *Ldet = nullptr, *cbuf = nullptr, *ubuf = nullptr;
    float2* Lxy = nullptr;  // interleaved (Lx, Ly)
    float* kval = nullptr;
    unsigned* hmax = nullptr;
    int* hist = nullptr;
    int* fallback = nullptr;
    uint32_t* bitmap = nullptr;
    int* work = nullptr;  // the descriptor pass's keypoint counter
    int* rowcnt = nullptr;
    int* rowoff = nullptr;
    // current build
    int n = 0, W = 0, H = 0;
    Geom geom{};
    size_t img_stride = 0;  // N * plane
    bool built = false, detected = false;
    bool edge_derivs = true;  // (Lx, Ly) of levels 0 and N−1 materialised by the last detect
    cudaStream_t last_stream = nullptr;
    // host path
    float* hin[2] = {nullptr, nullptr};
    kaze_keypoint* hkps[2] = {nullptr, nullptr};
    int* hcnt[2] = {nullptr, nullptr};
    float* hdesc[2] = {nullptr, nullptr};
    int* pinned_counts = nullptr;  // 2 * max_batch
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_cnt[2] = {}, ev_d2h[2] = {};
    // descriptor texture objects over the Lxy planes, [max_batch][N], one immutable table per image size: a
    // captured graph bakes the device pointer of its size's table, so a table is never rewritten; it is destroyed
    // only together with every graph of its size (LRU beyond kMaxTexTables sizes)
    struct TexTable {
        int W, H;
        std::vector<cudaTextureObject_t> texs;
        cudaTextureObject_t* d = nullptr;
        uint64_t used = 0;
    };
    std::vector<TexTable> tex_tables;
    // profiling
    bool prof = false;
    // CUDA graphs of whole chunks (build + detect + describe), keyed by everything a replay bakes in
    struct GraphKey {
        const void *img, *kps, *cnt, *desc;
        int n, w, h;
        int64_t pitch;
        cudaStream_t s;
        int part = 7;  // steps captured: 1 build, 2 detect, 4 describe
        bool operator==(const GraphKey& o) const {
            return img == o.img && kps == o.kps && cnt == o.cnt && desc == o.desc && n == o.n && w == o.w &&
                   h == o.h && pitch == o.pitch && s == o.s && part == o.part;
        }
    };
    struct GraphEntry {
        GraphKey key;
        cudaGraphExec_t exec;
        int64_t nk;
        uint64_t used;
    };
    std::vector<GraphEntry> graphs;
    std::vector<GraphKey> seen;
    uint64_t tick = 0;
    cudaStream_t s_cap = nullptr;
    // overlapped multi-chunk extraction: the descriptor pass of chunk j on a side stream, concurrent with the
    // scale space of chunk j+1 (s_side for direct runs, s_cap2 inside captures); per-chunk events
    cudaStream_t s_side = nullptr, s_cap2 = nullptr;
    std::vector<cudaEvent_t> ovl_ev;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    int64_t launches = 0;
    std::string err;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

cudaEvent_t get_event(kaze_ctx* c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Wraps one kernel launch: counts it and, when profiling, brackets it with events on its stream.
struct Launch {
    kaze_ctx* c;
    int kc;
    double bytes;
    cudaStream_t s;
    int nk;  // kernels launched inside this scope
    cudaEvent_t e0 = nullptr;
    Launch(kaze_ctx* c_, int kc_, double bytes_, cudaStream_t s_, int nk_ = 1)
        : c(c_), kc(kc_), bytes(bytes_), s(s_), nk(nk_) {
        if (c->prof) {
            e0 = get_event(c);
            cudaEventRecord(e0, s);
        }
    }
    ~Launch() {
        c->launches += nk;
        if (c->prof) {
            cudaEvent_t e1 = get_event(c);
            cudaEventRecord(e1, s);
            c->recs.push_back({kc, e0, e1, bytes, nk});
        }
    }
};

kaze_status cuda_fail(kaze_ctx* c, cudaError_t e, const char* where) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
    if (c) c->err = buf;
    return KAZE_ERR_CUDA;
}

#define KZ_CHECK_LAUNCH(ctx, where)                              \
    do {                                                         \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
    } while (0)

#define KZ_CUDA(ctx, call)                                        \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call);  \
    } while (0)

GaussTaps make_taps(double sigma) {
    GaussTaps t{};
    int r = (int)std::ceil(3.0 * sigma);
    if (r < 1) r = 1;
    t.r = r;
    double w[2 * kMaxGaussR + 1], s = 0.0;
    for (int i = -r; i <= r; ++i) {
        w[i + r] = std::exp(-(double)i * i / (2.0 * sigma * sigma));
        s += w[i + r];
    }
    for (int i = 0; i <= 2 * r; ++i) t.w[i] = (float)(w[i] / s);
    return t;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// One FED cycle of total time T (Eq. 5; A20, A21), as the product computes it:
//  * n = the smallest integer with τ_max·n(n+1)/3 >= T (the sum of Eq. 5's n steps is τ_max·n(n+1)/3);
//  * τ_j = q·τ_max / (2cos²(π(2j+1)/(4n+2))), j = 0..n−1, with q = T / (τ_max·n(n+1)/3) so the cycle ends at T;
//  * execution order j_m = (κ·m) mod n, κ coprime to n, minimising max_m max_μ|Π_{l<=m}(1 − τ_{j_l}μ)| ·
//    max_μ|Π_{l>m}(1 − τ_{j_l}μ)| over μ on 1025 points of [0, 8] (the spectrum of the 5-point operator with
//    c <= 1); ties → the smallest κ.  In fp32 the natural (increasing) order amplifies rounding by ~1e12 at
//    n = 29; this order keeps the cycle at the rounding level of a single step.
std::vector<float> fed_cycle(double T, double tau_max) {
    int n = 1;
    while (tau_max * n * (n + 1) / 3.0 < T) ++n;
    const double q = T / (tau_max * n * (n + 1) / 3.0);
    std::vector<double> tau(n);
    for (int j = 0; j < n; ++j) {
        const double cj = std::cos(M_PI * (2.0 * j + 1.0) / (4.0 * n + 2.0));
        tau[j] = q * tau_max / (2.0 * cj * cj);
    }
    auto gcd = [](int a, int b) {
        while (b) {
            const int r = a % b;
            a = b;
            b = r;
        }
        return a;
    };
    constexpr int kMu = 1025;
    int best = 1;
    double best_g = INFINITY;
    std::vector<double> fwd(n), bwd(n + 1);
    for (int kap = 1; kap < std::max(n, 2); ++kap) {
        if (gcd(kap, n) != 1) continue;
        std::fill(fwd.begin(), fwd.end(), 0.0);
        std::fill(bwd.begin(), bwd.end(), 0.0);
        bwd[n] = 1.0;
        for (int u = 0; u < kMu; ++u) {
            const double mu = 8.0 * u / (kMu - 1);
            double pf = 1.0, pb = 1.0;
            for (int m = 0; m < n; ++m) {
                pf *= 1.0 - tau[(size_t)((long)kap * m % n)] * mu;
                fwd[m] = std::max(fwd[m], std::fabs(pf));
                const int mb = n - 1 - m;
                pb *= 1.0 - tau[(size_t)((long)kap * mb % n)] * mu;
                bwd[mb] = std::max(bwd[mb], std::fabs(pb));
            }
        }
        double gk = 0.0;
        for (int m = 0; m < n; ++m) gk = std::max(gk, fwd[m] * bwd[m + 1]);
        if (gk < best_g) {
            best_g = gk;
            best = kap;
        }
    }
    std::vector<float> out(n);
    for (int m = 0; m < n; ++m) out[m] = (float)tau[(size_t)((long)best * m % n)];
    return out;
}

kaze_status validate_params(const kaze_params* p) {
    if (!p) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->octaves < 1 || p->sublevels < 1 || p->octaves * p->sublevels > kMaxLevels) return KAZE_ERR_INVALID_ARGUMENT;
    if (!(p->sigma0 > 0) || p->sigma0 > kMaxGaussR / 3.0) return KAZE_ERR_INVALID_ARGUMENT;
    if (!(p->k_percentile > 0 && p->k_percentile < 1)) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->k_bins < 1 || p->k_bins > kMaxBins) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->diffusivity < 1 || p->diffusivity > 3) return KAZE_ERR_INVALID_ARGUMENT;
    if (!(p->threshold >= 0)) return KAZE_ERR_INVALID_ARGUMENT;
    if (std::isnan(p->edge_ratio) || std::isnan(p->k_override)) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->max_keypoints < 1 || p->ori_windows < 1 || p->ori_windows > 64) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->max_batch < 1 || p->max_batch > kMaxBatch) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->max_width < 32 || p->max_height < 32) return KAZE_ERR_IMAGE_TOO_SMALL;
    if (p->max_width > 8192 || p->max_height > 8192) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->scheme != KAZE_SCHEME_AOS && p->scheme != KAZE_SCHEME_FED) return KAZE_ERR_INVALID_ARGUMENT;
    if (p->scheme == KAZE_SCHEME_FED && !(p->tau_max > 0 && p->tau_max <= 0.25)) return KAZE_ERR_INVALID_ARGUMENT;
    return KAZE_OK;
}

void free_arena(kaze_ctx* c) {
    void* ptrs[] = {c->Lt, c->Lxy, c->Ldet, c->cbuf, c->ubuf, c->kval, c->hmax, c->hist, c->fallback,
                    c->bitmap, c->rowcnt, c->rowoff, c->work, c->hin[0], c->hin[1], c->hkps[0], c->hkps[1],
                    c->hcnt[0], c->hcnt[1], c->hdesc[0], c->hdesc[1]};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (c->pinned_counts) cudaFreeHost(c->pinned_counts);
    for (auto& tt : c->tex_tables) {
        for (auto t : tt.texs) cudaDestroyTextureObject(t);
        if (tt.d) cudaFree(tt.d);
    }
    c->tex_tables.clear();
}

// Plane size in floats: pitch x H rounded to 128 floats, so every (image, level) plane of the interleaved float2
// derivative array starts 1024-byte aligned (texture base alignment for the descriptor's filtered fetches).
size_t plane_of(int W, int H) { return ((size_t)round_up(W, 32) * H + 127) / 128 * 128; }

// ---- the three steps, on one chunk of n <= max_batch images ----
void set_geometry(kaze_ctx* c, int n, int w, int h) {
    c->n = n;
    c->W = w;
    c->H = h;
    c->geom.W = w;
    c->geom.H = h;
    c->geom.P = round_up(w, 32);
    c->geom.plane = plane_of(w, h);
    c->img_stride = (size_t)c->N * c->geom.plane;
}

// Step 1 (P:L255-260 with the AOS solver of Eq. 4): prefilter → k → N−1 × {conductivity, AOS columns, AOS rows}.
kaze_status do_build(kaze_ctx* c, const float* d_imgs, int n, int w, int h, int64_t pitch, cudaStream_t s) {
    const int N = c->N;
    set_geometry(c, n, w, h);
    c->built = false;
    c->detected = false;
    Geom g = c->geom;  // g.rev: the conductivity and AOS passes alternate their image order (see below)
    const size_t SL = c->img_stride, SP = g.plane;  // pyramid stride, scratch stride
    const double px = (double)w * h * n;
    {
        Launch L(c, KC_PREFILTER, 8.0 * px, s);
        launch_prefilter(d_imgs, pitch, (size_t)pitch * h, c->Lt, SL, g, n, c->g0, s);
    }
    KZ_CHECK_LAUNCH(c, "prefilter");
    const bool estimate = !(c->p.k_override > 0);
    if (estimate) {
        KZ_CUDA(c, cudaMemsetAsync(c->hmax, 0, sizeof(unsigned) * n, s));
        KZ_CUDA(c, cudaMemsetAsync(c->hist, 0, sizeof(int) * (size_t)n * c->p.k_bins, s));
        {
            Launch L(c, KC_GRAD_L1, 8.0 * px, s);
            launch_cond(c->Lt, SL, c->cbuf, SP, g, n, c->g1, 0, c->p.diffusivity, c->kval, c->hmax, s);
        }
        KZ_CHECK_LAUNCH(c, "grad_l1");
        {
            Launch L(c, KC_KHIST, 4.0 * px, s);
            launch_khist(c->cbuf, SP, g, n, c->p.k_bins, c->hmax, c->hist, s);
        }
        KZ_CHECK_LAUNCH(c, "k_hist");
    }
    {
        Launch L(c, KC_KFINAL, 0.0, s);
        launch_kfinal(c->hist, c->p.k_bins, c->hmax, n, c->p.k_percentile, c->p.k_override, c->kval, c->fallback, s);
    }
    KZ_CHECK_LAUNCH(c, "k_final");
    // Level loop.  KAZE_BUILD_SUB=k (diagnostic knob) runs it on sub-batches of k images, image-major, so that a
    // sub-batch's c, U and L_i planes can stay in L2 between the passes of a level.
    static const int sub = tune_knob("KAZE_BUILD_SUB", 0);
    const int sb = sub > 0 ? std::min(sub, n) : n;
    // Pass order: each conductivity / column / row pass walks the batch in the opposite image order to the pass
    // before it, so it starts on the images whose planes the previous pass touched last (still L2-resident);
    // KAZE_ALTERNATE=0 keeps every pass ascending.
    static const int alternate = tune_knob("KAZE_ALTERNATE", 1);
    int pass = 1;
    auto next_order = [&]() {
        g.rev = alternate ? (pass & 1) : 0;
        ++pass;
    };
    for (int b0 = 0; b0 < n; b0 += sb) {
        const int m = std::min(sb, n - b0);
        const double mpx = (double)w * h * m;
        float* Lt = c->Lt + (size_t)b0 * SL;
        float* cb = c->cbuf + (size_t)b0 * SP;
        float* ub = c->ubuf + (size_t)b0 * SP;
        const float* kv = c->kval + b0;
        for (int i = 1; i < N; ++i) {
            const float* prev = Lt + (size_t)(i - 1) * g.plane;
            float* cur = Lt + (size_t)i * g.plane;
            {   // level 1 too: recomputing |∇(G1∗L0)|² in the conductivity pass beats converting the stored |∇|²
                // (measured 1.45 vs 2.6 ms per 256-image step)
                Launch L(c, KC_COND, 8.0 * mpx, s);
                next_order();
                launch_cond(prev, SL, cb, SP, g, m, c->g1, 1, c->p.diffusivity, kv, nullptr, s);
            }
            KZ_CHECK_LAUNCH(c, "cond");
            if (c->p.scheme == KAZE_SCHEME_FED) {  // one FED cycle, K <= kFedMaxK steps per launch (A20, A21)
                const std::vector<float>& taus = c->fed[i];
                const int ns = (int)taus.size(), nl = (ns + kFedMaxK - 1) / kFedMaxK;
                int done = 0;
                for (int j = 0; j < nl; ++j) {
                    const int k = (ns - done + (nl - j) - 1) / (nl - j);
                    FedTaus ft{};
                    for (int q = 0; q < k; ++q) ft.t[q] = taus[done + q];
                    // ping-pong so that the last launch writes L_i: launch j writes cur iff nl-1-j is even
                    float* dst = ((nl - 1 - j) % 2 == 0) ? cur : ub;
                    const float* src = j == 0 ? prev : (((nl - j) % 2 == 0) ? cur : ub);
                    const size_t s_src = j == 0 ? SL : (src == cur ? SL : SP), s_dst = dst == cur ? SL : SP;
                    {
                        Launch L(c, KC_FED, 12.0 * mpx, s);
                        g.rev = 0;
                        launch_fed_steps(src, s_src, cb, SP, dst, s_dst, g, m, ft, k, s);
                    }
                    KZ_CHECK_LAUNCH(c, "fed");
                    done += k;
                }
                continue;
            }
            const float tau = (float)(c->t[i] - c->t[i - 1]);
            {   // U = column solves (ubuf holds U)
                Launch L(c, KC_AOS_COLS, 12.0 * mpx, s);
                next_order();
                if (!launch_aos_cols(prev, cb, ub, Strides{SL, SP, 0, SP}, g, m, tau, s))
                    return KAZE_ERR_INVALID_ARGUMENT;
            }
            KZ_CHECK_LAUNCH(c, "aos_cols");
            {   // L_i = ½(U + V), V = row solves
                Launch L(c, KC_AOS_ROWS, 16.0 * mpx, s);
                next_order();
                if (!launch_aos_rows(prev, cb, ub, cur, Strides{SL, SP, SP, SL}, g, m, tau, s))
                    return KAZE_ERR_INVALID_ARGUMENT;
            }
            KZ_CHECK_LAUNCH(c, "aos_rows");
        }
    }
    c->built = true;
    c->last_stream = s;
    return KAZE_OK;
}

// Step 2 (Eq. 8).
kaze_status do_detect(kaze_ctx* c, kaze_keypoint* d_kps, int32_t* d_counts, cudaStream_t s) {
    const int N = c->N, n = c->n;
    const Geom g = c->geom;
    const double px = (double)g.W * g.H * n;
    {   // Hessian (Eq. 8), all levels of all images in one fused launch (two chain passes for steps > 32)
        static const int fused = tune_knob("KAZE_HESS_FUSED", 1);
        if (fused) {
            const int keep = (c->p.flags & KAZE_FLAG_ALL_DERIVATIVES) ? 1 : 0;
            // 16 B/px per level; the first and last level store no (Lx, Ly) unless asked: 8 B/px there
            Launch L(c, KC_HESSIAN, (keep ? 16.0 * N : 16.0 * N - 16.0) * px, s, 1);
            c->edge_derivs = keep != 0;
            if (!launch_hess_fused(c->Lt, c->Lxy, c->Ldet, c->img_stride, g, n, c->lt, keep, s)) {
                launch_hess_first(c->Lt, c->Lxy, c->img_stride, g, n, c->lt, s);
                launch_hess_det(c->Lxy, c->Ldet, c->img_stride, g, n, c->lt, s);
                L.bytes = 24.0 * px * N;
                L.nk = 2;
                c->edge_derivs = true;
            }
        } else {
            c->edge_derivs = true;
            Launch L(c, KC_HESSIAN, 24.0 * px * N, s, 2);
            launch_hess_first(c->Lt, c->Lxy, c->img_stride, g, n, c->lt, s);
            launch_hess_det(c->Lxy, c->Ldet, c->img_stride, g, n, c->lt, s);
        }
    }
    KZ_CHECK_LAUNCH(c, "hessian");
    if (N < 3) {
        KZ_CUDA(c, cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * n, s));
    } else {
        DetectParams dp{(float)c->p.threshold, (float)c->p.edge_ratio, c->p.max_keypoints,
                        (c->p.flags & KAZE_FLAG_EXACT_WINDOW) ? 1 : 0, (c->p.flags & KAZE_FLAG_REFINE_3D) ? 1 : 0};
        {
            Launch L(c, KC_NMS_MARK, 4.0 * px * N, s, 2);  // nms_mark (1 or 2 launches) + rowcount
            L.nk = launch_nms_mark(c->Ldet, c->img_stride, g, n, c->lt, dp, c->bitmap, c->rowcnt, s);
        }
        KZ_CHECK_LAUNCH(c, "nms_mark");
        const int R = (N - 2) * g.H;
        {
            Launch L(c, KC_KP_SCAN, 8.0 * R * n, s);
            launch_kp_scan(c->rowcnt, R, n, c->rowoff, d_counts, s);
        }
        KZ_CHECK_LAUNCH(c, "kp_scan");
        {
            Launch L(c, KC_KP_EMIT, 0.0, s);
            launch_kp_emit(c->Ldet, c->img_stride, g, n, c->lt, dp, c->bitmap, c->rowcnt, c->rowoff, d_kps, s);
        }
        KZ_CHECK_LAUNCH(c, "kp_emit");
    }
    c->detected = true;
    c->last_stream = s;
    return KAZE_OK;
}

// Texture objects (bilinear filtering, clamped addressing, unnormalised coordinates) over every (image, level)
// Lxy plane of the current geometry, for the descriptor's 576 filtered samples per keypoint.  One table per image
// size, built once (synchronous upload, before any capture) and immutable afterwards.
constexpr size_t kMaxTexTables = 16;

void drop_graphs_of_size(kaze_ctx* c, int w, int h);

kaze_status ensure_textures(kaze_ctx* c, const cudaTextureObject_t** out) {
    for (auto& tt : c->tex_tables)
        if (tt.W == c->W && tt.H == c->H) {
            tt.used = ++c->tick;
            *out = tt.d;
            return KAZE_OK;
        }
    if (c->tex_tables.size() >= kMaxTexTables) {  // evict the least recently used size and its graphs
        auto lru = std::min_element(c->tex_tables.begin(), c->tex_tables.end(),
                                    [](const auto& a, const auto& b) { return a.used < b.used; });
        KZ_CUDA(c, cudaDeviceSynchronize());  // a launched graph or kernel may still sample it
        drop_graphs_of_size(c, lru->W, lru->H);
        for (auto t : lru->texs) cudaDestroyTextureObject(t);
        if (lru->d) cudaFree(lru->d);
        c->tex_tables.erase(lru);
    }
    const int B = c->p.max_batch, N = c->N;
    kaze_ctx::TexTable tt;
    tt.W = c->W;
    tt.H = c->H;
    tt.texs.assign((size_t)B * N, 0);
    auto cleanup = [&]() {
        for (auto t : tt.texs)
            if (t) cudaDestroyTextureObject(t);
        if (tt.d) cudaFree(tt.d);
    };
    if (cudaMalloc(&tt.d, sizeof(cudaTextureObject_t) * B * N) != cudaSuccess) {
        cudaGetLastError();
        tt.d = nullptr;
        cleanup();
        return KAZE_ERR_OOM;
    }
    for (int b = 0; b < B; ++b)
        for (int l = 0; l < N; ++l) {
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypePitch2D;
            rd.res.pitch2D.devPtr = c->Lxy + (size_t)b * c->img_stride + (size_t)l * c->geom.plane;
            rd.res.pitch2D.desc = cudaCreateChannelDesc<float2>();
            rd.res.pitch2D.width = c->W;
            rd.res.pitch2D.height = c->H;
            rd.res.pitch2D.pitchInBytes = sizeof(float2) * c->geom.P;
            cudaTextureDesc td{};
            td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
            td.filterMode = cudaFilterModeLinear;
            td.readMode = cudaReadModeElementType;
            td.normalizedCoords = 0;
            const cudaError_t e = cudaCreateTextureObject(&tt.texs[(size_t)b * N + l], &rd, &td, nullptr);
            if (e != cudaSuccess) {
                cleanup();
                return cuda_fail(c, e, "cudaCreateTextureObject");
            }
        }
    const cudaError_t e = cudaMemcpy(tt.d, tt.texs.data(), sizeof(cudaTextureObject_t) * B * N, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(c, e, "texture table upload");
    }
    tt.used = ++c->tick;
    c->tex_tables.push_back(std::move(tt));
    *out = c->tex_tables.back().d;
    return KAZE_OK;
}

// Step 3.
kaze_status do_describe(kaze_ctx* c, kaze_keypoint* d_kps, const int32_t* d_counts, float* d_desc, cudaStream_t s,
                        bool overlapped = false) {
    const cudaTextureObject_t* texs = nullptr;
    kaze_status st = ensure_textures(c, &texs);
    if (st != KAZE_OK) return st;
    {
        Launch L(c, KC_DESCRIBE, 0.0, s);
        const int lo = c->edge_derivs ? 0 : 1, hi = c->edge_derivs ? c->N - 1 : c->N - 2;  // sampleable levels
        static const int dyn = tune_knob("KAZE_DESC_DYN", 1);
        if (dyn) KZ_CUDA(c, cudaMemsetAsync(c->work, 0, sizeof(int), s));
        launch_describe(c->Lxy, texs, c->img_stride, c->geom, c->n, c->N, lo, hi, dyn ? c->work : nullptr,
                        overlapped ? 1 : 0, d_kps, d_counts, c->p.max_keypoints,
                        d_desc, c->p.ori_windows, (c->p.flags & KAZE_FLAG_KEEP_ANGLE) ? 1 : 0, s);
    }
    KZ_CHECK_LAUNCH(c, "describe");
    c->last_stream = s;
    return KAZE_OK;
}

// One chunk of m <= max_batch images through the three steps, directly or as a CUDA graph: a chunk key seen for
// the first time runs directly (which also settles every lazily initialised kernel attribute and the texture
// objects), the second time it is captured on the context's private stream, and from then on its graph is
// replayed on the caller's stream.  Graphs are per key (pointers, sizes, stream); at most kMaxGraphs are kept.
constexpr size_t kMaxGraphs = 96;

// `part` selects the steps (1 build, 2 detect, 4 describe; the describe of an overlapped schedule passes 8 too, for
// the smaller persistent grid).
kaze_status run_chunk_direct(kaze_ctx* c, const float* img, int m, int w, int h, int64_t pitch, kaze_keypoint* kps,
                             int32_t* cnt, float* desc, cudaStream_t s, int part = 7) {
    kaze_status st = KAZE_OK;
    if (part & 1) st = do_build(c, img, m, w, h, pitch, s);
    if (st != KAZE_OK) return st;
    if (part & 2) st = do_detect(c, kps, cnt, s);
    if (st != KAZE_OK) return st;
    if (part & 4) st = do_describe(c, kps, cnt, desc, s, (part & 8) != 0);
    return st;
}

kaze_status run_chunk(kaze_ctx* c, const float* img, int m, int w, int h, int64_t pitch, kaze_keypoint* kps,
                      int32_t* cnt, float* desc, cudaStream_t s, int part = 7) {
    if (c->prof || (c->p.flags & KAZE_FLAG_NO_GRAPHS))
        return run_chunk_direct(c, img, m, w, h, pitch, kps, cnt, desc, s, part);
    const kaze_ctx::GraphKey key{img, kps, cnt, desc, m, w, h, pitch, s, part};
    for (auto& ge : c->graphs)
        if (ge.key == key) {
            set_geometry(c, m, w, h);
            KZ_CUDA(c, cudaGraphLaunch(ge.exec, s));
            c->launches += ge.nk;
            ge.used = ++c->tick;
            c->built = c->detected = true;
            c->last_stream = s;
            return KAZE_OK;
        }
    bool again = false;
    for (auto& k : c->seen) again |= (k == key);
    if (!again) {
        if (c->seen.size() >= 4 * kMaxGraphs) c->seen.erase(c->seen.begin());
        c->seen.push_back(key);
        return run_chunk_direct(c, img, m, w, h, pitch, kps, cnt, desc, s, part);
    }
    if (!c->s_cap) KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_cap, cudaStreamNonBlocking));
    set_geometry(c, m, w, h);
    const cudaTextureObject_t* texs = nullptr;
    kaze_status st = ensure_textures(c, &texs);  // host-side setup (synchronous copies) must precede the capture
    if (st != KAZE_OK) return st;
    // the capture stream must not start before the caller's prior work when the graph is launched; a graph
    // launched on s is ordered after s's prior work by the launch itself, so the capture needs no dependency
    const int64_t l0 = c->launches;
    KZ_CUDA(c, cudaStreamBeginCapture(c->s_cap, cudaStreamCaptureModeThreadLocal));
    pdl_set_capturing(true);
    st = run_chunk_direct(c, img, m, w, h, pitch, kps, cnt, desc, c->s_cap, part);
    pdl_set_capturing(false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->s_cap, &graph);
    if (st != KAZE_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ec != cudaSuccess) {
        c->err = std::string("graph capture: ") + cudaGetErrorString(ec);
        return KAZE_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        c->err = std::string("graph instantiate: ") + cudaGetErrorString(ei);
        return KAZE_ERR_CUDA;
    }
    const int64_t nk = c->launches - l0;
    c->launches = l0;  // the capture launched nothing
    if (c->graphs.size() >= kMaxGraphs) {
        auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                    [](const auto& a, const auto& b) { return a.used < b.used; });
        cudaGraphExecDestroy(lru->exec);
        c->graphs.erase(lru);
    }
    c->graphs.push_back({key, exec, nk, ++c->tick});
    KZ_CUDA(c, cudaGraphLaunch(exec, s));
    c->launches += nk;
    c->built = c->detected = true;
    c->last_stream = s;
    return KAZE_OK;
}

void drop_graphs_of_size(kaze_ctx* c, int w, int h) {
    for (size_t i = 0; i < c->graphs.size();) {
        if (c->graphs[i].key.w == w && c->graphs[i].key.h == h) {
            cudaGraphExecDestroy(c->graphs[i].exec);
            c->graphs.erase(c->graphs.begin() + (long)i);
        } else {
            ++i;
        }
    }
    for (size_t i = 0; i < c->seen.size();) {
        if (c->seen[i].w == w && c->seen[i].h == h) c->seen.erase(c->seen.begin() + (long)i);
        else ++i;
    }
}

// Several chunks with the descriptor pass overlapped: describe(j) runs on `side` while build(j+1) runs on `main`;
// detect(j+1) rewrites the Lxy pyramid that describe(j) samples, so it waits for describe(j).  Every other buffer a
// describe reads (keypoints, counts of its own chunk, the texture table) is untouched by the next chunk.  The
// describe pass is gather/TEX-bound while the scale-space passes are L1/latency-bound, so they share the SMs.
kaze_status run_chunks_overlapped(kaze_ctx* c, const float* img, int n, int w, int h, int64_t pitch,
                                  kaze_keypoint* kps, int32_t* cnt, float* desc, cudaStream_t main_s,
                                  cudaStream_t side_s) {
    const int B = c->p.max_batch;
    const size_t cap = (size_t)c->p.max_keypoints;
    // (A quarter-size last chunk, whose descriptor pass nothing overlaps, measured no change here: 1836.7 / 1832.0 vs
    // 1835.8 / 1832.9 img/s; the host path keeps it for its result copies.)
    const int nch = (n + B - 1) / B;
    while ((int)c->ovl_ev.size() < 2 * nch) {
        cudaEvent_t e;
        KZ_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ovl_ev.push_back(e);
    }
    for (int j = 0; j < nch; ++j) {
        const int i0 = j * B, m = std::min(B, n - i0);
        kaze_status st = do_build(c, img + (size_t)i0 * pitch * h, m, w, h, pitch, main_s);
        if (st != KAZE_OK) return st;
        if (j > 0) KZ_CUDA(c, cudaStreamWaitEvent(main_s, c->ovl_ev[2 * (j - 1) + 1], 0));
        st = do_detect(c, kps + (size_t)i0 * cap, cnt + i0, main_s);
        if (st != KAZE_OK) return st;
        KZ_CUDA(c, cudaEventRecord(c->ovl_ev[2 * j], main_s));
        KZ_CUDA(c, cudaStreamWaitEvent(side_s, c->ovl_ev[2 * j], 0));
        st = do_describe(c, kps + (size_t)i0 * cap, cnt + i0, desc + (size_t)i0 * cap * 64, side_s, true);
        if (st != KAZE_OK) return st;
        KZ_CUDA(c, cudaEventRecord(c->ovl_ev[2 * j + 1], side_s));
    }
    KZ_CUDA(c, cudaStreamWaitEvent(main_s, c->ovl_ev[2 * (nch - 1) + 1], 0));
    c->last_stream = main_s;
    return KAZE_OK;
}

// The whole call (n > max_batch) as one overlapped CUDA graph, by the same first-direct / second-capture /
// then-replay rule as run_chunk (the key's n > max_batch keeps it apart from the chunk graphs).
kaze_status run_overlapped(kaze_ctx* c, const float* img, int n, int w, int h, int64_t pitch, kaze_keypoint* kps,
                           int32_t* cnt, float* desc, cudaStream_t s) {
    if (!c->s_side) KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking));
    const kaze_ctx::GraphKey key{img, kps, cnt, desc, n, w, h, pitch, s};
    for (auto& ge : c->graphs)
        if (ge.key == key) {
            set_geometry(c, std::min(c->p.max_batch, n - (n - 1) / c->p.max_batch * c->p.max_batch), w, h);
            KZ_CUDA(c, cudaGraphLaunch(ge.exec, s));
            c->launches += ge.nk;
            ge.used = ++c->tick;
            c->built = c->detected = true;
            c->last_stream = s;
            return KAZE_OK;
        }
    bool again = false;
    for (auto& k : c->seen) again |= (k == key);
    if (!again || (c->p.flags & KAZE_FLAG_NO_GRAPHS)) {
        if (!again) {
            if (c->seen.size() >= 4 * kMaxGraphs) c->seen.erase(c->seen.begin());
            c->seen.push_back(key);
        }
        return run_chunks_overlapped(c, img, n, w, h, pitch, kps, cnt, desc, s, c->s_side);
    }
    if (!c->s_cap) KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_cap, cudaStreamNonBlocking));
    if (!c->s_cap2) KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_cap2, cudaStreamNonBlocking));
    set_geometry(c, c->p.max_batch, w, h);
    const cudaTextureObject_t* texs = nullptr;
    kaze_status st = ensure_textures(c, &texs);  // host-side setup before the capture
    if (st != KAZE_OK) return st;
    const int64_t l0 = c->launches;
    KZ_CUDA(c, cudaStreamBeginCapture(c->s_cap, cudaStreamCaptureModeThreadLocal));
    pdl_set_capturing(true);
    st = run_chunks_overlapped(c, img, n, w, h, pitch, kps, cnt, desc, c->s_cap, c->s_cap2);
    pdl_set_capturing(false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->s_cap, &graph);
    if (st != KAZE_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ec != cudaSuccess) {
        c->err = std::string("graph capture: ") + cudaGetErrorString(ec);
        return KAZE_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        c->err = std::string("graph instantiate: ") + cudaGetErrorString(ei);
        return KAZE_ERR_CUDA;
    }
    const int64_t nk = c->launches - l0;
    c->launches = l0;
    if (c->graphs.size() >= kMaxGraphs) {
        auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                    [](const auto& a, const auto& b) { return a.used < b.used; });
        cudaGraphExecDestroy(lru->exec);
        c->graphs.erase(lru);
    }
    c->graphs.push_back({key, exec, nk, ++c->tick});
    KZ_CUDA(c, cudaGraphLaunch(exec, s));
    c->launches += nk;
    c->built = c->detected = true;
    c->last_stream = s;
    return KAZE_OK;
}

kaze_status check_dims(const kaze_ctx* c, int n, int w, int h, int64_t pitch) {
    if (n < 1 || n > c->p.max_batch) return KAZE_ERR_INVALID_ARGUMENT;
    if (w < 32 || h < 32 || w > c->p.max_width || h > c->p.max_height) return KAZE_ERR_IMAGE_TOO_SMALL;
    if (pitch < w) return KAZE_ERR_INVALID_ARGUMENT;
    if (c->sigma[c->N - 1] > 0.5 * std::min(w, h)) return KAZE_ERR_IMAGE_TOO_SMALL;  // S:L222 as validation (A4)
    return KAZE_OK;
}

kaze_status ensure_host_path(kaze_ctx* c) {
    if (c->s_h2d) return KAZE_OK;
    const int B = c->p.max_batch;
    const size_t cap = (size_t)c->p.max_keypoints;
    for (int b = 0; b < 2; ++b) {
        if (cudaMalloc(&c->hin[b], sizeof(float) * c->plane_max * B) != cudaSuccess) return KAZE_ERR_OOM;
        if (cudaMalloc(&c->hkps[b], sizeof(kaze_keypoint) * cap * B) != cudaSuccess) return KAZE_ERR_OOM;
        if (cudaMalloc(&c->hcnt[b], sizeof(int) * B) != cudaSuccess) return KAZE_ERR_OOM;
        if (cudaMalloc(&c->hdesc[b], sizeof(float) * 64 * cap * B) != cudaSuccess) return KAZE_ERR_OOM;
        KZ_CUDA(c, cudaEventCreateWithFlags(&c->ev_h2d[b], cudaEventDisableTiming));
        KZ_CUDA(c, cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming));
        KZ_CUDA(c, cudaEventCreateWithFlags(&c->ev_cnt[b], cudaEventDisableTiming));
        KZ_CUDA(c, cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming));
    }
    if (cudaMallocHost(&c->pinned_counts, sizeof(int) * 2 * B) != cudaSuccess) return KAZE_ERR_OOM;
    KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    return KAZE_OK;
}

}  // namespace

// =====================================================================================================================
extern "C" {

kaze_status kaze_default_params(kaze_params* p) {
    if (!p) return KAZE_ERR_INVALID_ARGUMENT;
    memset(p, 0, sizeof(*p));
    p->max_width = 1920;
    p->max_height = 1200;
    p->max_batch = 1;
    p->octaves = 4;
    p->sublevels = 4;
    p->sigma0 = 1.6;
    p->k_percentile = 0.7;
    p->k_bins = 300;
    p->diffusivity = 2;
    p->k_override = 0.0;
    p->threshold = 1e-3;
    p->edge_ratio = 10.0;
    p->max_keypoints = 65536;
    p->ori_windows = 42;
    p->flags = 0;
    p->scheme = KAZE_SCHEME_AOS;
    p->tau_max = 0.25;
    return KAZE_OK;
}

int32_t kaze_abi_version(void) { return KAZE_ABI_VERSION; }

kaze_status kaze_create(const kaze_params* p, int device, kaze_ctx** out) {
    if (!out) return KAZE_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    kaze_status st = validate_params(p);
    if (st != KAZE_OK) return st;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return KAZE_ERR_CUDA;
    DeviceGuard guard(device);
    kaze_ctx* c = new kaze_ctx();
    c->p = *p;
    c->device = device;
    c->N = p->octaves * p->sublevels;
    // Eq. 6 read as σ_i = σ0·2^{o + s/S} (A3), Eq. 7 t_i = σ_i²/2, s_i = max(1, floor(σ_i + ½)) (A9)
    for (int o = 0; o < p->octaves; ++o)
        for (int sl = 0; sl < p->sublevels; ++sl) {
            const int i = o * p->sublevels + sl;
            c->sigma[i] = p->sigma0 * std::pow(2.0, (double)o + (double)sl / p->sublevels);
            c->t[i] = 0.5 * c->sigma[i] * c->sigma[i];
            const int stp = (int)std::floor(c->sigma[i] + 0.5);
            c->step[i] = stp < 1 ? 1 : stp;
            c->lt.step[i] = c->step[i];
            c->lt.sigma[i] = (float)c->sigma[i];
        }
    if (p->scheme == KAZE_SCHEME_FED) {
        c->fed.resize(c->N);
        for (int i = 1; i < c->N; ++i) c->fed[i] = fed_cycle(c->t[i] - c->t[i - 1], p->tau_max);
    }
    c->lt.n = c->N;
    c->lt.S = p->sublevels;
    c->g0 = make_taps(p->sigma0);
    c->g1 = make_taps(1.0);
    c->Pmax = round_up(p->max_width, 32);
    c->plane_max = plane_of(p->max_width, p->max_height);  // >= every build's plane (see plane_of)
    const size_t B = p->max_batch, N = c->N;
    const size_t pyr = sizeof(float) * c->plane_max * N * B;
    const int words = nms_words(p->max_width);
    const size_t rows = (size_t)(N > 2 ? N - 2 : 1) * p->max_height * B;
    bool ok = cudaMalloc(&c->Lt, pyr) == cudaSuccess && cudaMalloc(&c->Lxy, 2 * pyr) == cudaSuccess &&
              cudaMalloc(&c->Ldet, pyr) == cudaSuccess &&
              cudaMalloc(&c->cbuf, sizeof(float) * c->plane_max * B) == cudaSuccess &&
              cudaMalloc(&c->ubuf, sizeof(float) * c->plane_max * B) == cudaSuccess &&
              cudaMalloc(&c->kval, sizeof(float) * B) == cudaSuccess &&
              cudaMalloc(&c->hmax, sizeof(unsigned) * B) == cudaSuccess &&
              cudaMalloc(&c->hist, sizeof(int) * B * p->k_bins) == cudaSuccess &&
              cudaMalloc(&c->fallback, sizeof(int) * B) == cudaSuccess &&
              cudaMalloc(&c->bitmap, sizeof(uint32_t) * rows * words) == cudaSuccess &&
              cudaMalloc(&c->rowcnt, sizeof(int) * rows) == cudaSuccess &&
              cudaMalloc(&c->rowoff, sizeof(int) * rows) == cudaSuccess &&
              cudaMalloc(&c->work, sizeof(int)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        free_arena(c);
        delete c;
        return KAZE_ERR_OOM;
    }
    cudaMemset(c->hist, 0, sizeof(int) * B * p->k_bins);
    cudaMemset(c->hmax, 0, sizeof(unsigned) * B);
    init_describe_tables();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        free_arena(c);
        delete c;
        return KAZE_ERR_CUDA;
    }
    *out = c;
    return KAZE_OK;
}

kaze_status kaze_destroy(kaze_ctx* c) {
    if (!c) return KAZE_OK;
    DeviceGuard guard(c->device);
    cudaDeviceSynchronize();
    for (auto& r : c->recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b) {
        if (c->ev_h2d[b]) cudaEventDestroy(c->ev_h2d[b]);
        if (c->ev_comp[b]) cudaEventDestroy(c->ev_comp[b]);
        if (c->ev_cnt[b]) cudaEventDestroy(c->ev_cnt[b]);
        if (c->ev_d2h[b]) cudaEventDestroy(c->ev_d2h[b]);
    }
    for (auto& ge : c->graphs) cudaGraphExecDestroy(ge.exec);
    for (auto e : c->ovl_ev) cudaEventDestroy(e);
    if (c->s_side) cudaStreamDestroy(c->s_side);
    if (c->s_cap2) cudaStreamDestroy(c->s_cap2);
    if (c->s_cap) cudaStreamDestroy(c->s_cap);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    free_arena(c);
    delete c;
    return KAZE_OK;
}

kaze_status kaze_build_scale_space(kaze_ctx* c, const float* d_imgs, int32_t n, int32_t w, int32_t h,
                                   int64_t pitch, void* stream) {
    if (!c || !d_imgs) return KAZE_ERR_INVALID_ARGUMENT;
    kaze_status st = check_dims(c, n, w, h, pitch);
    if (st != KAZE_OK) return st;
    DeviceGuard guard(c->device);
    return do_build(c, d_imgs, n, w, h, pitch, (cudaStream_t)stream);
}

kaze_status kaze_detect(kaze_ctx* c, kaze_keypoint* d_kps, int32_t* d_counts, void* stream) {
    if (!c || !d_kps || !d_counts) return KAZE_ERR_INVALID_ARGUMENT;
    if (!c->built) return KAZE_ERR_STATE;
    DeviceGuard guard(c->device);
    return do_detect(c, d_kps, d_counts, (cudaStream_t)stream);
}

kaze_status kaze_describe(kaze_ctx* c, kaze_keypoint* d_kps, const int32_t* d_counts, float* d_desc, void* stream) {
    if (!c || !d_kps || !d_counts || !d_desc) return KAZE_ERR_INVALID_ARGUMENT;
    if (!c->built) return KAZE_ERR_STATE;
    DeviceGuard guard(c->device);
    return do_describe(c, d_kps, d_counts, d_desc, (cudaStream_t)stream);
}

kaze_status kaze_extract(kaze_ctx* c, const float* d_imgs, int32_t n, int32_t w, int32_t h, int64_t pitch,
                         kaze_keypoint* d_kps, int32_t* d_counts, float* d_desc, void* stream) {
    if (!c || (n > 0 && (!d_imgs || !d_kps || !d_counts || !d_desc)) || n < 0) return KAZE_ERR_INVALID_ARGUMENT;
    if (n == 0) return KAZE_OK;
    kaze_status st = check_dims(c, 1, w, h, pitch);
    if (st != KAZE_OK) return st;
    DeviceGuard guard(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cap = (size_t)c->p.max_keypoints;
    // several chunks: the descriptor pass of each chunk overlaps the next chunk's scale space (KAZE_OVERLAP=0: one
    // chunk after the other); profiling keeps the sequential direct launches so per-kernel times stay separable
    static const int overlap = tune_knob("KAZE_OVERLAP", 1);
    if (overlap && n > c->p.max_batch && !c->prof)
        return run_overlapped(c, d_imgs, n, w, h, pitch, d_kps, d_counts, d_desc, s);
    for (int i0 = 0; i0 < n; i0 += c->p.max_batch) {
        const int m = n - i0 < c->p.max_batch ? n - i0 : c->p.max_batch;
        st = run_chunk(c, d_imgs + (size_t)i0 * pitch * h, m, w, h, pitch, d_kps + i0 * cap, d_counts + i0,
                       d_desc + i0 * cap * 64, s);
        if (st != KAZE_OK) return st;
    }
    return KAZE_OK;
}

kaze_status kaze_extract_host(kaze_ctx* c, const float* h_imgs, int32_t n, int32_t w, int32_t h, int64_t pitch,
                              kaze_keypoint* h_kps, int32_t* h_counts, float* h_desc, void* stream) {
    if (!c || n < 0 || (n > 0 && (!h_imgs || !h_kps || !h_counts))) return KAZE_ERR_INVALID_ARGUMENT;
    if (n == 0) return KAZE_OK;
    kaze_status st = check_dims(c, 1, w, h, pitch);
    if (st != KAZE_OK) return st;
    DeviceGuard guard(c->device);
    st = ensure_host_path(c);
    if (st != KAZE_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int B = c->p.max_batch;
    const size_t cap = (size_t)c->p.max_keypoints;
    const int P = round_up(w, 32);
    // Chunk boundaries: when there is more than one chunk, the first holds a quarter of max_batch, so the upload the
    // first build must wait for (nothing overlaps it) is short; so does the last (KAZE_HOST_TAIL), whose descriptor
    // pass and result copies nothing overlaps either; the others are full, a remainder before the last.
    static const int small_tail = tune_knob("KAZE_HOST_TAIL", 1);
    std::vector<int> cb{0};
    const int quarter = std::max(1, B / 4);
    const int tail = (small_tail && n > B + quarter) ? quarter : 0;
    if (n > B) cb.push_back(quarter);
    while (cb.back() < n - tail) cb.push_back(std::min(n - tail, cb.back() + B));
    if (tail) cb.push_back(n);
    const int nchunks = (int)cb.size() - 1;
    // Make the context's copy streams start after prior work on the caller's stream.
    KZ_CUDA(c, cudaEventRecord(c->ev_comp[0], s));
    KZ_CUDA(c, cudaStreamWaitEvent(c->s_h2d, c->ev_comp[0], 0));
    // KAZE_TRACE_HOST=1: timing events around every chunk's H2D, compute and D2H, printed to stderr (diagnostics)
    static const int trace = tune_knob("KAZE_TRACE_HOST", 0);
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) -> int {
        if (!trace) return -1;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.push_back(e);
        return (int)tev.size() - 1;
    };
    std::vector<int> tmarks;
    const int t0mark = mark(s);
    // Overlap (as kaze_extract, KAZE_OVERLAP): chunk j's describe runs on the side stream while chunk j+1's scale
    // space runs on s; detect(j+1) waits for describe(j) (Lxy), and chunk j's keypoint/descriptor copies for its
    // describe (ev_desc[b]).  The parts run as separate graphs (keyed by part).
    static const int overlap = tune_knob("KAZE_OVERLAP", 1);
    const bool ovl = overlap && nchunks > 1 && !c->prof;
    if (ovl && !c->s_side) KZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking));
    while (ovl && (int)c->ovl_ev.size() < 4) {
        cudaEvent_t e;
        KZ_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ovl_ev.push_back(e);
    }
    // ovl_ev[b]: describe of the chunk in buffer b done; ovl_ev[2 + b]: its detect done
    auto finalize = [&](int j) -> kaze_status {
        const int b = j & 1, i0 = cb[j], m = cb[j + 1] - cb[j];
        KZ_CUDA(c, cudaEventSynchronize(c->ev_cnt[b]));
        KZ_CUDA(c, cudaStreamWaitEvent(c->s_d2h, ovl ? c->ovl_ev[b] : c->ev_cnt[b], 0));
        tmarks.push_back(mark(c->s_d2h));
        const int* cnt = c->pinned_counts + b * B;
        for (int i = 0; i < m; ++i) {
            h_counts[i0 + i] = cnt[i];
            const size_t nk = (size_t)(cnt[i] < (int)cap ? cnt[i] : (int)cap);
            if (nk == 0) continue;
            KZ_CUDA(c, cudaMemcpyAsync(h_kps + (size_t)(i0 + i) * cap, c->hkps[b] + (size_t)i * cap,
                                       nk * sizeof(kaze_keypoint), cudaMemcpyDeviceToHost, c->s_d2h));
            if (h_desc)
                KZ_CUDA(c, cudaMemcpyAsync(h_desc + (size_t)(i0 + i) * cap * 64, c->hdesc[b] + (size_t)i * cap * 64,
                                           nk * 64 * sizeof(float), cudaMemcpyDeviceToHost, c->s_d2h));
        }
        KZ_CUDA(c, cudaEventRecord(c->ev_d2h[b], c->s_d2h));
        tmarks.push_back(mark(c->s_d2h));
        return KAZE_OK;
    };
    for (int j = 0; j < nchunks; ++j) {
        const int b = j & 1, i0 = cb[j], m = cb[j + 1] - cb[j];
        // H2D of chunk j into buffer b, once the compute of chunk j-2 stopped reading it
        if (j >= 2) KZ_CUDA(c, cudaStreamWaitEvent(c->s_h2d, c->ev_comp[b], 0));
        tmarks.push_back(mark(c->s_h2d));
        if (pitch == P)  // rows already at the device pitch: one linear copy
            KZ_CUDA(c, cudaMemcpyAsync(c->hin[b], h_imgs + (size_t)i0 * pitch * h, sizeof(float) * P * h * m,
                                       cudaMemcpyHostToDevice, c->s_h2d));
        else
            KZ_CUDA(c, cudaMemcpy2DAsync(c->hin[b], sizeof(float) * P, h_imgs + (size_t)i0 * pitch * h,
                                         sizeof(float) * pitch, sizeof(float) * w, (size_t)m * h,
                                         cudaMemcpyHostToDevice, c->s_h2d));
        KZ_CUDA(c, cudaEventRecord(c->ev_h2d[b], c->s_h2d));
        KZ_CUDA(c, cudaStreamWaitEvent(s, c->ev_h2d[b], 0));
        if (j >= 2) KZ_CUDA(c, cudaStreamWaitEvent(s, c->ev_d2h[b], 0));
        tmarks.push_back(mark(c->s_h2d));
        tmarks.push_back(mark(s));
        if (ovl) {
            st = run_chunk(c, c->hin[b], m, w, h, P, c->hkps[b], c->hcnt[b], c->hdesc[b], s, 1);
            if (st != KAZE_OK) return st;
            KZ_CUDA(c, cudaEventRecord(c->ev_comp[b], s));  // input buffer b is free once the build is done
            if (j >= 1) KZ_CUDA(c, cudaStreamWaitEvent(s, c->ovl_ev[b ^ 1], 0));  // describe(j-1) done with Lxy
            st = run_chunk(c, c->hin[b], m, w, h, P, c->hkps[b], c->hcnt[b], c->hdesc[b], s, 2);
            if (st != KAZE_OK) return st;
            KZ_CUDA(c, cudaEventRecord(c->ovl_ev[2 + b], s));
            KZ_CUDA(c, cudaStreamWaitEvent(c->s_side, c->ovl_ev[2 + b], 0));
            st = run_chunk(c, c->hin[b], m, w, h, P, c->hkps[b], c->hcnt[b], c->hdesc[b], c->s_side, 4 | 8);
            if (st != KAZE_OK) return st;
            KZ_CUDA(c, cudaEventRecord(c->ovl_ev[b], c->s_side));
        } else {
            st = run_chunk(c, c->hin[b], m, w, h, P, c->hkps[b], c->hcnt[b], c->hdesc[b], s);
            if (st != KAZE_OK) return st;
            KZ_CUDA(c, cudaEventRecord(c->ev_comp[b], s));  // input buffer b is free once the chunk is done
        }
        tmarks.push_back(mark(s));
        KZ_CUDA(c, cudaMemcpyAsync(c->pinned_counts + b * B, c->hcnt[b], sizeof(int) * m, cudaMemcpyDeviceToHost, s));
        KZ_CUDA(c, cudaEventRecord(c->ev_cnt[b], s));
        // (the D2H stream waits for this chunk inside finalize(j), right before its copies: a wait enqueued here
        // would hold chunk j-1's copies, enqueued next, behind chunk j's compute — measured 12 ms per 128 images)
        if (j >= 1) {
            st = finalize(j - 1);
            if (st != KAZE_OK) return st;
        }
    }
    st = finalize(nchunks - 1);
    if (st != KAZE_OK) return st;
    if (ovl) KZ_CUDA(c, cudaStreamWaitEvent(s, c->ovl_ev[(nchunks - 1) & 1], 0));  // s ends after the last describe
    KZ_CUDA(c, cudaStreamSynchronize(c->s_d2h));
    if (trace) {
        cudaDeviceSynchronize();
        // per chunk j: h2d start/end, compute start/end (in order of recording); d2h start/end of chunk j-1
        for (size_t q = 0; q < tmarks.size(); ++q) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tev[t0mark], tev[tmarks[q]]);
            fprintf(stderr, "%s%.2f", q ? " " : "trace:", ms);
        }
        fprintf(stderr, "\n");
        for (auto e : tev) cudaEventDestroy(e);
    }
    return KAZE_OK;
}

kaze_status kaze_get_k(kaze_ctx* c, float* h_k, int32_t* h_fallback) {
    if (!c || !h_k) return KAZE_ERR_INVALID_ARGUMENT;
    if (!c->built) return KAZE_ERR_STATE;
    DeviceGuard guard(c->device);
    KZ_CUDA(c, cudaStreamSynchronize(c->last_stream));
    KZ_CUDA(c, cudaMemcpy(h_k, c->kval, sizeof(float) * c->n, cudaMemcpyDeviceToHost));
    if (h_fallback) KZ_CUDA(c, cudaMemcpy(h_fallback, c->fallback, sizeof(int) * c->n, cudaMemcpyDeviceToHost));
    return KAZE_OK;
}

static kaze_status plane_ptr(kaze_ctx* c, int32_t img, int32_t level, int32_t which, float** out) {
    if (!c->built) return KAZE_ERR_STATE;
    if (img < 0 || img >= c->n) return KAZE_ERR_INVALID_ARGUMENT;
    if (which != KAZE_PLANE_COND && (level < 0 || level >= c->N)) return KAZE_ERR_INVALID_ARGUMENT;
    const size_t off = (size_t)img * c->img_stride + (size_t)level * c->geom.plane;
    switch (which) {
        case KAZE_PLANE_LT: *out = c->Lt + off; break;
        case KAZE_PLANE_LX:
        case KAZE_PLANE_LY: *out = reinterpret_cast<float*>(c->Lxy + off); break;
        case KAZE_PLANE_LDET: *out = c->Ldet + off; break;
        case KAZE_PLANE_COND: *out = c->cbuf + (size_t)img * c->geom.plane; break;
        default: return KAZE_ERR_INVALID_ARGUMENT;
    }
    return KAZE_OK;
}

kaze_status kaze_get_level(kaze_ctx* c, int32_t img, int32_t level, int32_t which, float* d_out, void* stream) {
    if (!c || !d_out) return KAZE_ERR_INVALID_ARGUMENT;
    if ((which == KAZE_PLANE_LX || which == KAZE_PLANE_LY) && (level == 0 || level == c->N - 1) && !c->edge_derivs)
        return KAZE_ERR_STATE;
    float* src = nullptr;
    kaze_status st = plane_ptr(c, img, level, which, &src);
    if (st != KAZE_OK) return st;
    DeviceGuard guard(c->device);
    if (which == KAZE_PLANE_LX || which == KAZE_PLANE_LY) {
        launch_component_copy(reinterpret_cast<float2*>(src), which == KAZE_PLANE_LY, d_out, 1, c->geom,
                              (cudaStream_t)stream);
        KZ_CHECK_LAUNCH(c, "get_level");
        return KAZE_OK;
    }
    KZ_CUDA(c, cudaMemcpy2DAsync(d_out, sizeof(float) * c->W, src, sizeof(float) * c->geom.P, sizeof(float) * c->W,
                                 c->H, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return KAZE_OK;
}

kaze_status kaze_set_level(kaze_ctx* c, int32_t img, int32_t level, int32_t which, const float* d_in, void* stream) {
    if (!c || !d_in) return KAZE_ERR_INVALID_ARGUMENT;
    float* dst = nullptr;
    kaze_status st = plane_ptr(c, img, level, which, &dst);
    if (st != KAZE_OK) return st;
    DeviceGuard guard(c->device);
    if (which == KAZE_PLANE_LX || which == KAZE_PLANE_LY) {
        launch_component_copy(reinterpret_cast<float2*>(dst), which == KAZE_PLANE_LY, const_cast<float*>(d_in), 0,
                              c->geom, (cudaStream_t)stream);
        KZ_CHECK_LAUNCH(c, "set_level");
        return KAZE_OK;
    }
    KZ_CUDA(c, cudaMemcpy2DAsync(dst, sizeof(float) * c->geom.P, d_in, sizeof(float) * c->W, sizeof(float) * c->W,
                                 c->H, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return KAZE_OK;
}

kaze_status kaze_set_profiling(kaze_ctx* c, int32_t enable) {
    if (!c) return KAZE_ERR_INVALID_ARGUMENT;
    c->prof = enable != 0;
    return KAZE_OK;
}

kaze_status kaze_reset_profile(kaze_ctx* c) {
    if (!c) return KAZE_ERR_INVALID_ARGUMENT;
    DeviceGuard guard(c->device);
    for (auto& r : c->recs) {
        c->pool.push_back(r.e0);
        c->pool.push_back(r.e1);
    }
    c->recs.clear();
    c->launches = 0;
    return KAZE_OK;
}

kaze_status kaze_get_profile(kaze_ctx* c, kaze_kernel_stat* out, int32_t cap, int32_t* n) {
    if (!c || !n || (cap > 0 && !out)) return KAZE_ERR_INVALID_ARGUMENT;
    DeviceGuard guard(c->device);
    KZ_CUDA(c, cudaDeviceSynchronize());
    kaze_kernel_stat acc[KC_COUNT];
    memset(acc, 0, sizeof(acc));
    for (int k = 0; k < KC_COUNT; ++k) snprintf(acc[k].name, sizeof(acc[k].name), "%s", kKernelNames[k]);
    for (auto& r : c->recs) {
        float ms = 0.f;
        KZ_CUDA(c, cudaEventElapsedTime(&ms, r.e0, r.e1));
        acc[r.kc].launches += r.nk;
        acc[r.kc].total_ms += ms;
        acc[r.kc].algo_bytes += r.bytes;
    }
    int m = 0;
    for (int k = 0; k < KC_COUNT; ++k) {
        if (acc[k].launches == 0) continue;
        if (m < cap) out[m] = acc[k];
        ++m;
    }
    *n = m;
    return KAZE_OK;
}

int64_t kaze_launch_count(const kaze_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"

namespace kz {
int tune_knob(const char* name, int def) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : def;
}
namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_smem_optin;  // (function, device) -> bytes set
std::map<int, int> g_sm_count;                              // device -> multiprocessor count
}  // namespace
bool ensure_smem_optin(const void* func, int bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& have = g_smem_optin[{func, dev}];
    if (have >= bytes) return true;
    if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    have = bytes;
    return true;
}
int device_sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_sm_count.find(dev);
    if (it != g_sm_count.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 1;
    g_sm_count[dev] = n;
    return n;
}
static thread_local bool g_capturing = false;
void pdl_set_capturing(bool on) { g_capturing = on; }
bool pdl_enabled() {
    // Measured (256-image step, graph replay): programmatic edges inside the captured graphs cost 160 -> 196 ms;
    // for direct launches they cut the 400x240 scale space from 0.258 to 0.174 ms.  So: direct launches only.
    static const int mode = tune_knob("KAZE_PDL", 1);
    return mode == 2 || (mode == 1 && !g_capturing);
}
}  // namespace kz

extern "C" {

kaze_status kaze_memory_footprint(const kaze_ctx* c, kaze_memory* out) {
    if (!c || !out) return KAZE_ERR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    const uint64_t B = c->p.max_batch, N = c->N, plane = sizeof(float) * c->plane_max;
    const uint64_t rows = (uint64_t)(N > 2 ? N - 2 : 1) * c->p.max_height * B;
    const uint64_t cap = (uint64_t)c->p.max_keypoints;
    out->evolution = plane * N * B;
    out->derivatives = 2 * plane * N * B;
    out->response = plane * N * B;
    out->scratch = 2 * plane * B;
    out->detector = sizeof(float) * B + sizeof(unsigned) * B + sizeof(int) * B * c->p.k_bins + sizeof(int) * B +
                    sizeof(uint32_t) * rows * nms_words(c->p.max_width) + 2 * sizeof(int) * rows + sizeof(int);
    out->textures = sizeof(cudaTextureObject_t) * B * N * (uint64_t)c->tex_tables.size();
    if (c->s_h2d) {
        out->host_path = 2 * (plane * B + sizeof(kaze_keypoint) * cap * B + sizeof(int) * B + sizeof(float) * 64 * cap * B);
        out->pinned_host = sizeof(int) * 2 * B;
    }
    out->total = out->evolution + out->derivatives + out->response + out->scratch + out->detector + out->textures +
                 out->host_path;
    return KAZE_OK;
}

size_t kaze_match_scratch_bytes(int32_t na, int32_t nb) {
    if (na < 0 || nb < 0) return 0;
    return match_scratch_bytes(na, nb);
}

kaze_status kaze_match(const float* d_a, int32_t na, const float* d_b, int32_t nb, float ratio, int32_t* d_match,
                       float* d_dist, void* d_scratch, size_t scratch_bytes, int32_t* d_stats, void* stream) {
    if (na < 0 || nb < 0 || !(ratio > 0.f && ratio <= 1.f)) return KAZE_ERR_INVALID_ARGUMENT;
    if ((na > 0 && (!d_a || !d_match)) || (nb > 0 && !d_b)) return KAZE_ERR_INVALID_ARGUMENT;
    if (na == 0) return KAZE_OK;
    if (!d_scratch || scratch_bytes < match_scratch_bytes(na, nb)) return KAZE_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(d_a) | reinterpret_cast<uintptr_t>(d_b) |
         reinterpret_cast<uintptr_t>(d_scratch)) & 15u)
        return KAZE_ERR_INVALID_ARGUMENT;
    const int rc = match_run(d_a, na, d_b, nb, ratio, d_match, d_dist, d_scratch, scratch_bytes, d_stats,
                             (cudaStream_t)stream);
    return rc == 0 ? KAZE_OK : KAZE_ERR_CUDA;
}

int32_t kaze_fed_cycle(double T, double tau_max, float* taus, int32_t cap) {
    if (!(T > 0) || !(tau_max > 0 && tau_max <= 0.25) || cap < 0 || (cap > 0 && !taus)) return KAZE_ERR_INVALID_ARGUMENT;
    const std::vector<float> t = fed_cycle(T, tau_max);
    for (int32_t j = 0; j < cap && j < (int32_t)t.size(); ++j) taus[j] = t[j];
    return (int32_t)t.size();
}


const char* kaze_status_string(kaze_status s) {
    switch (s) {
        case KAZE_OK: return "ok";
        case KAZE_ERR_INVALID_ARGUMENT: return "invalid argument";
        case KAZE_ERR_IMAGE_TOO_SMALL: return "image too small (or larger than the context maxima)";
        case KAZE_ERR_CAPACITY: return "capacity";
        case KAZE_ERR_STATE: return "call out of order (build -> detect -> describe)";
        case KAZE_ERR_CUDA: return "CUDA error";
        case KAZE_ERR_OOM: return "device out of memory";
    }
    return "unknown status";
}

const char* kaze_last_error(const kaze_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

}  // extern "C"
