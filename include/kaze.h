/*
 * kaze.h — C ABI of the B200-native KAZE hot path (arXiv 1706.06750, "GPGPU Acceleration of the
 * KAZE Image Feature Extraction Algorithm").  Implementation: libkaze_b200.so (sm_100a CUDA).
 *
 * Citations: "P:Lnnn" = PAPER.md line nnn; "A<n>" = reading n in DESIGN.md §3 (where the paper is
 * silent or garbled).  The method, in the paper's three steps:
 *   1. nonlinear scale space: Gaussian prefilter σ0, contrast k from the gradient histogram
 *      (A7), Perona–Malik g2 conductivity (Eqs. 2-3), and one semi-implicit
 *      AOS step of Eq. 4 per evolution time t_i = σ_i²/2 (Eqs. 6-7, A1-A3) — or, with
 *      scheme = KAZE_SCHEME_FED, one FED cycle of Eq. 5 per level (A20-A21)
 *      → kaze_build_scale_space;
 *   2. scale-normalised Hessian determinant (Eq. 8, A9-A10), 3x3x3 extrema above the
 *      threshold, edge test (Eqs. 9-12) and 2-D sub-pixel fit → kaze_detect;
 *   3. dominant orientation and 64-D M-SURF descriptor → kaze_describe.
 *
 * Conventions (all entry points):
 *  - Plain pointers only.  "d_" pointers are CUDA device memory on the context's device, owned by
 *    the caller; "h_" pointers are host memory owned by the caller (pinned memory recommended for
 *    kaze_extract_host).  Images are fp32, row-major, values in [0, 1] (A17), with a row pitch in
 *    ELEMENTS (>= width).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Compute entry points
 *    enqueue work on it and return without synchronising; argument errors are detected and returned
 *    synchronously before anything is enqueued; asynchronous CUDA faults surface as KAZE_ERR_CUDA on
 *    a later call (text via kaze_last_error).
 *  - A context belongs to one device and is not thread-safe; distinct contexts may run concurrently.
 *  - The context owns all scratch (pyramid, histograms, k, bitmaps), allocated once at kaze_create for
 *    max_batch images of at most max_width x max_height.
 */
#ifndef KAZE_B200_H
#define KAZE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KAZE_ABI_VERSION 3

typedef struct kaze_ctx kaze_ctx;

typedef enum {
    KAZE_OK = 0,
    KAZE_ERR_INVALID_ARGUMENT = -1, /* bad parameter value, null pointer, n > max_batch, ...      */
    KAZE_ERR_IMAGE_TOO_SMALL = -2,  /* min(w, h) < 32, σ_{N−1} > min(w, h)/2, or w/h above maxima */
    KAZE_ERR_CAPACITY = -3,         /* reserved: capacity overflow is reported through d_counts    */
    KAZE_ERR_STATE = -4,            /* detect before build, describe before detect                 */
    KAZE_ERR_CUDA = -5,             /* CUDA runtime error (see kaze_last_error)                    */
    KAZE_ERR_OOM = -6               /* device allocation failed at kaze_create                     */
} kaze_status;

/* Parameters.  Defaults (kaze_default_params) follow the KAZE defaults of BASELINE configs[1]. */
typedef struct {
    int32_t max_width, max_height, max_batch; /* arena sizing, fixed at kaze_create (>= 32, >= 1) */
    int32_t octaves;       /* O >= 1, default 4 (Eq. 6)                              */
    int32_t sublevels;     /* S >= 1, default 4; N = O*S levels, all at full resolution  */
    double  sigma0;        /* σ0 > 0, default 1.6 (Eq. 6; prefilter P:L255)                       */
    double  k_percentile;  /* in (0, 1), default 0.7 (A7)                             */
    int32_t k_bins;        /* 1..4096, default 300 (A7)                                           */
    int32_t diffusivity;   /* 2 = g2 (default), 1 = g1 (Eq. 3), 3 = Weickert (A24)    */
    double  k_override;    /* <= 0: estimate k per image; > 0: use this k for every image         */
    double  threshold;     /* >= 0, default 1e-3: keep Ldet > threshold (A11)         */
    double  edge_ratio;    /* r of Eq. 12, default 10; <= 0 disables the edge test   */
    int32_t max_keypoints; /* per-image capacity of the keypoint / descriptor outputs, >= 1       */
    int32_t ori_windows;   /* sliding-window centres for the orientation, default 42, 1..64 (A14) */
    int32_t flags;         /* KAZE_FLAG_* below                                                   */
    int32_t scheme;        /* KAZE_SCHEME_AOS (default; Eq. 4, A1) or KAZE_SCHEME_FED (Eq. 5, A20) */
    double  tau_max;       /* FED: stability bound of one explicit step, in (0, 0.25], default 0.25 */
} kaze_params;

/* Scale-space solver (kaze_params.scheme). */
#define KAZE_SCHEME_AOS 0  /* one semi-implicit AOS step of Eq. 4 per level                  */
#define KAZE_SCHEME_FED 1  /* one FED cycle per level: n explicit steps with Eq. 5 step sizes scaled to
                              reach t_i exactly, n = min{n : τ_max n(n+1)/3 >= t_i − t_{i−1}}, in the
                              κ-cycle order of A21                                          */

/* kaze_describe uses the angles already stored in d_kps instead of computing them (stage-isolated
 * parity tests with pinned angles). */
#define KAZE_FLAG_KEEP_ANGLE 1
/* Detector variants.  EXACT_WINDOW: the paper's exact procedure — besides its 3x3 ring at
 * level i, a keypoint must exceed every in-image response of the (2r_i+1)² window at levels i−1 and i+1,
 * r_i = max(1, floor(s_i/2)) (A22).  REFINE_3D: quadratic fit in (x, y, level) from the
 * 3x3x3 block instead of the 2-D fit; σ = σ_i·2^{δs/S} (A23). */
#define KAZE_FLAG_EXACT_WINDOW 2
#define KAZE_FLAG_REFINE_3D 4
/* kaze_extract / kaze_extract_host replay each (inputs, outputs, sizes, stream) chunk they have seen twice as one
 * CUDA graph (captured on a private stream, launched on the caller's); this flag disables that (every kernel is
 * launched directly).  Profiling (kaze_set_profiling) also launches directly. */
#define KAZE_FLAG_NO_GRAPHS 8
/* Materialise (Lx, Ly) of the first and last level too.  Those two levels carry no keypoints (A11), so their first
 * derivatives feed only their own Ldet, which the fused Hessian pass forms on chip; by default they are not stored
 * and kaze_get_level(KAZE_PLANE_LX / LY) of level 0 or N−1 returns KAZE_ERR_STATE. */
#define KAZE_FLAG_ALL_DERIVATIVES 16

/* 32-byte keypoint (P:L212-214 sub-pixel position; D4 of SURVEY). */
typedef struct {
    float   x, y;          /* sub-pixel position in pixels, full input resolution               */
    float   sigma;         /* σ_i of the detection level                                         */
    float   response;      /* Ldet at the integer extremum                                       */
    float   angle;         /* dominant orientation in [0, 2π), written by kaze_describe          */
    int32_t level;         /* evolution level i in 1..N-2                                        */
    int16_t octave;        /* o = i / S                                                          */
    int16_t sublevel;      /* s = i % S                                                          */
    int32_t flags;         /* bit 0: degenerate orientation (all samples zero); descriptor = 0   */
} kaze_keypoint;

/* Which pyramid plane kaze_get_level / kaze_set_level address. */
typedef enum {
    KAZE_PLANE_LT = 0,     /* evolution image L_i (level 0..N-1)                                 */
    KAZE_PLANE_LX = 1,     /* s_i-normalised first derivative s·∂x L_i                            */
    KAZE_PLANE_LY = 2,     /* s_i-normalised first derivative s·∂y L_i                            */
    KAZE_PLANE_LDET = 3,   /* scale-normalised Hessian determinant (Eq. 8)                        */
    KAZE_PLANE_COND = 4    /* conductivity c_i of the LAST built level (level argument ignored)  */
} kaze_plane;

/* Fills *p with the defaults (max_width = 1920, max_height = 1200, max_batch = 1,
 * max_keypoints = 65536).  Errors: INVALID_ARGUMENT if p is NULL. */
kaze_status kaze_default_params(kaze_params* p);

/* Creates a context on CUDA device `device` and allocates its arena.  Errors: INVALID_ARGUMENT
 * (null pointer, out-of-range parameter), IMAGE_TOO_SMALL (max_width/max_height < 32), OOM, CUDA. */
kaze_status kaze_create(const kaze_params* p, int device, kaze_ctx** out);

/* Frees the context and its arena (synchronises the device first).  NULL is accepted. */
kaze_status kaze_destroy(kaze_ctx* ctx);

/* Step 1: nonlinear scale space for n images d_imgs[n][h][pitch] (n <= max_batch, 32 <= w <=
 * max_width, 32 <= h <= max_height, pitch >= w).  Levels stay in the context until the next build.
 * The largest scale must fit the image: σ_{N−1} = σ0·2^{O−1+(S−1)/S} <= min(w, h)/2 (SPEC's "levels whose σ_i
 * exceeds min(W,H)/2 are dropped", read as validation), else IMAGE_TOO_SMALL — e.g. the
 * default O = S = 4 (σ_15 ≈ 21.5) needs min(w, h) >= 43.
 * Errors: INVALID_ARGUMENT, IMAGE_TOO_SMALL, CUDA. */
kaze_status kaze_build_scale_space(kaze_ctx* ctx, const float* d_imgs, int32_t n, int32_t w, int32_t h,
                                   int64_t pitch_elems, void* stream);

/* Step 2: Hessian response of every level, extrema, edge test, sub-pixel fit.  Writes image j's
 * keypoints to d_kps[j * max_keypoints + 0 .. min(count_j, max_keypoints)) in (level, y, x) order and
 * the TRUE count to d_counts[j] (count > max_keypoints signals truncation).  d_kps: n*max_keypoints
 * entries, d_counts: n entries (device).  Errors: INVALID_ARGUMENT, STATE (no build), CUDA. */
kaze_status kaze_detect(kaze_ctx* ctx, kaze_keypoint* d_kps, int32_t* d_counts, void* stream);

/* Step 3: orientation (unless KAZE_FLAG_KEEP_ANGLE; angle and flags written into d_kps) and 64-D
 * descriptors d_desc[j * max_keypoints + k][64] for k < min(d_counts[j], max_keypoints), over the flat
 * list of all keypoints of all levels and images.  Degenerate descriptors are zero.
 * d_counts may be the array kaze_detect wrote, or caller-supplied (stage-isolated use).  A keypoint whose
 * level is outside 0..N−1, or is 0 or N−1 while those levels' (Lx, Ly) are not materialised (no detector output
 * lies there; KAZE_FLAG_ALL_DERIVATIVES stores them), gets a zero descriptor, angle 0 and flags bit 0 set.
 * Errors: INVALID_ARGUMENT, STATE (no build), CUDA. */
kaze_status kaze_describe(kaze_ctx* ctx, kaze_keypoint* d_kps, const int32_t* d_counts, float* d_desc,
                          void* stream);

/* Convenience: build + detect + describe for n images (any n >= 0; processed in chunks of
 * max_batch).  Outputs are indexed by image as in kaze_detect / kaze_describe.  With more than one
 * chunk, each chunk's describe runs on a context-private side stream concurrently with the next
 * chunk's build (the next detect waits for it); the call still completes in `stream` order.  Unless
 * KAZE_FLAG_NO_GRAPHS is set (or profiling is on, which also runs the chunks one after the other), a
 * call whose (d_imgs, d_kps, d_counts, d_desc, n, w, h, pitch, stream) key has been seen twice is
 * replayed as one CUDA graph captured on context-private streams (the graph bakes in those pointers;
 * up to 96 keys are cached, least recently used evicted); results are bit-identical to direct
 * launches.  The call is asynchronous on `stream` like the stage entry points.  Errors: as the stage
 * entry points, plus CUDA for a failed capture or instantiation. */
kaze_status kaze_extract(kaze_ctx* ctx, const float* d_imgs, int32_t n, int32_t w, int32_t h,
                         int64_t pitch_elems, kaze_keypoint* d_kps, int32_t* d_counts, float* d_desc,
                         void* stream);

/* End-to-end from HOST buffers: h_imgs[n][h][pitch] → h_kps[n][max_keypoints], h_counts[n],
 * h_desc[n][max_keypoints][64] (h_desc may be NULL to skip descriptor download).  Copies run on
 * context-owned streams overlapped with compute (double-buffered chunks of at most max_batch images;
 * with more than one chunk the first holds max_batch/4 images, so the upload nothing can overlap is
 * short, and beyond max_batch + max_batch/4 images so does the last, whose descriptor pass and result
 * copies nothing can overlap; describes overlap the next chunk as in kaze_extract); the call returns
 * after everything has landed in host memory.  `stream` orders the work after prior work on it.
 * Errors: as kaze_extract. */
kaze_status kaze_extract_host(kaze_ctx* ctx, const float* h_imgs, int32_t n, int32_t w, int32_t h,
                              int64_t pitch_elems, kaze_keypoint* h_kps, int32_t* h_counts, float* h_desc,
                              void* stream);

/* ---- test / diagnostic entry points ---- */

/* Contrast factor of each image of the last build (host copies; synchronises the stream of the last
 * build).  h_k, h_fallback: max_batch entries (h_fallback may be NULL). */
kaze_status kaze_get_k(kaze_ctx* ctx, float* h_k, int32_t* h_fallback);

/* Copies plane `which` of level `level` of image `img` (h x w, tightly packed) to/from d_buf.
 * Errors: INVALID_ARGUMENT (range), STATE (nothing built; or LX / LY of level 0 or N−1 without
 * KAZE_FLAG_ALL_DERIVATIVES), CUDA. */
kaze_status kaze_get_level(kaze_ctx* ctx, int32_t img, int32_t level, int32_t which, float* d_out, void* stream);
kaze_status kaze_set_level(kaze_ctx* ctx, int32_t img, int32_t level, int32_t which, const float* d_in, void* stream);

/* Per-kernel-class device timing with CUDA events on the launching stream (off by default).
 * kaze_get_profile synchronises, then reports, for each kernel class, launches, summed device ms and
 * summed ALGORITHMIC bytes.  Returns the number of classes in *n. */
typedef struct {
    char    name[32];
    int64_t launches;
    double  total_ms;
    double  algo_bytes;
} kaze_kernel_stat;
kaze_status kaze_set_profiling(kaze_ctx* ctx, int32_t enable);
kaze_status kaze_get_profile(kaze_ctx* ctx, kaze_kernel_stat* out, int32_t cap, int32_t* n);
kaze_status kaze_reset_profile(kaze_ctx* ctx);
/* Number of kernels this context has launched since creation (or the last reset). */
int64_t kaze_launch_count(const kaze_ctx* ctx);

/* Device memory the context holds, by role (the paper's memory-footprint study, P:L424-437,
 * Fig. "Memory foot print").  Byte counts are exactly the sizes the context passed to cudaMalloc; they depend
 * only on kaze_params (max_width, max_height, max_batch, octaves, sublevels, k_bins, max_keypoints), not on
 * the images built since.  The paper's "scratch images L_step" are `scratch` here.  Errors:
 * INVALID_ARGUMENT if ctx or out is NULL. */
typedef struct {
    uint64_t evolution;   /* L_i pyramid: max_batch x N planes (pitch x height fp32, 512 B aligned)   */
    uint64_t derivatives; /* interleaved (Lx, Ly) pyramid, float2                                      */
    uint64_t response;    /* Ldet pyramid                                                               */
    uint64_t scratch;     /* conductivity c and the AOS column result U (or FED ping-pong), per image */
    uint64_t detector;    /* contrast k, hmax, histograms, fallback flags, candidate bitmap, row scans */
    uint64_t textures;    /* descriptor texture-object table (allocated at the first kaze_describe)     */
    uint64_t host_path;   /* kaze_extract_host staging (device side, 2 buffers; 0 until first used)    */
    uint64_t pinned_host; /* pinned host bytes of kaze_extract_host (0 until first used)               */
    uint64_t total;       /* sum of the device fields                                                   */
} kaze_memory;
kaze_status kaze_memory_footprint(const kaze_ctx* ctx, kaze_memory* out);

/* ---- descriptor matching (reading A25) — context-free ----
 * Brute-force L2 matching of d_a[na][64] against d_b[nb][64] (fp32, row-major, 16-byte aligned, device):
 * for each a its nearest and second-nearest non-degenerate (nonzero) b, ties → lower index; kept iff
 * d1 < ratio·d2 (d2 = ∞ with fewer than two candidates) and a is b's nearest non-degenerate a (cross-check).
 * d_match[na] ← b or −1; d_dist[na] (may be NULL) ← d1 (−1 if no candidate); d_stats (may be NULL, device
 * int32[2]) ← [number of matches, rows that needed the exact fallback scan].  The dot products run on the
 * tensor cores (fp16 operands, fp32 accumulation); candidates are re-ranked with exact fp32 distances and the
 * result is certified against the fp16 error bound, else the row is rescanned exactly, so the decisions are
 * the exact fp32 ones.  d_scratch: kaze_match_scratch_bytes(na, nb) bytes of device memory owned by the
 * caller.  Asynchronous on `stream`.  Errors: INVALID_ARGUMENT (counts < 0, ratio outside (0, 1], null or
 * misaligned pointers, scratch too small), CUDA. */
size_t kaze_match_scratch_bytes(int32_t na, int32_t nb);
kaze_status kaze_match(const float* d_a, int32_t na, const float* d_b, int32_t nb, float ratio, int32_t* d_match,
                       float* d_dist, void* d_scratch, size_t scratch_bytes, int32_t* d_stats, void* stream);

/* Host-only: the FED cycle the context runs for a level transition of total time T (Eq. 5, A20) —
 * step sizes in execution order (A21) written to taus[0 .. min(n, cap)); returns n (> 0), or
 * KAZE_ERR_INVALID_ARGUMENT for T <= 0, tau_max outside (0, 0.25], or taus == NULL with cap > 0. */
int32_t kaze_fed_cycle(double T, double tau_max, float* taus, int32_t cap);

const char* kaze_status_string(kaze_status s);
const char* kaze_last_error(const kaze_ctx* ctx);
int32_t kaze_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KAZE_B200_H */
