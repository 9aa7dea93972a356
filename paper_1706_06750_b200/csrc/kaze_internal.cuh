// kaze_internal.cuh — shared declarations of the sm_100a KAZE kernels and their launchers.
// Product code: nothing here is shared with oracle/ (DESIGN.md §2).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kaze.h"

namespace kz {

constexpr int kMaxLevels = 64;
constexpr int kMaxGaussR = 24;   // sigma0 <= 8
constexpr int kMaxBins = 4096;
constexpr int kMaxBatch = 1024;

// Plane geometry of one build: W x H pixels, pitch P floats (multiple of 32), plane = P * H.
struct Geom {
    int W, H, P;
    int rev;  // image order of a batched launch (cond / AOS passes): 0 ascending, 1 descending — consecutive passes
              // alternate, so a pass starts on the images the previous one touched last (still in L2)
    size_t plane;
};
// Image of batch slot z (of n) under the launch's order.
__device__ __forceinline__ int batch_image(int z, int n, const Geom& g) { return g.rev ? n - 1 - z : z; }

struct GaussTaps {
    int r;
    float w[2 * kMaxGaussR + 1];
};

struct LevelTable {          // per-level scalars passed by value to whole-pyramid kernels
    int n;                   // number of levels N
    int S;                   // sublevels
    int step[kMaxLevels];    // s_i (Eq. 8 derivative step, A9)
    float sigma[kMaxLevels]; // σ_i
};

// ---- programmatic dependent launch (PDL) ----
// Every kernel of the path starts with KZ_PDL_PROLOGUE(): griddepcontrol.wait blocks until the preceding kernel in
// the stream has completed and its writes are visible (a no-op without a programmatic dependency), then
// launch_dependents lets the NEXT kernel's CTAs be scheduled as this grid's CTAs retire, so launch latency and
// ramp-up overlap this kernel's tail.  kz_launch sets the programmatic-serialization attribute (knob KAZE_PDL=0
// turns it off).  Because every kernel waits before touching memory, dependencies stay transitive.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define KZ_PDL_PROLOGUE() \
    do {                  \
        kz::pdl_wait();   \
        kz::pdl_trigger(); \
    } while (0)

// PDL mode (knob KAZE_PDL): 0 off; 1 for direct launches only (not inside captured CUDA graphs); 2 always.
bool pdl_enabled();
void pdl_set_capturing(bool on);

template <typename... KArgs, typename... Args>
inline void kz_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Debug/tuning knob read once from the environment (A/B runs only; the defaults are the measured best).
int tune_knob(const char* name, int def);

// Function attributes are per device and kaze.h lets contexts on different devices run concurrently: opt `func`
// into `bytes` of dynamic shared memory on the CURRENT device (once per (function, device), thread safe; a larger
// request raises it).  Returns false if the driver refuses.
bool ensure_smem_optin(const void* func, int bytes);
// Tiled fp32 tensor map of `rank` dimensions (strides in bytes for dimensions 1..rank-1, element strides 1, no
// swizzle, out-of-bounds elements zero-filled) through cuTensorMapEncodeTiled (runtime driver entry point, no libcuda
// link).  Returns false if the encoder is unavailable or rejects the map.
bool encode_f32_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                    const cuuint32_t* box);
// Multiprocessor count of the current device (cached per device).
int device_sm_count();

// ---- stencil.cu ----
void launch_prefilter(const float* img, int64_t in_pitch, size_t in_img_stride, float* L0,
                      size_t out_img_stride, Geom g, int nimg, const GaussTaps& t, cudaStream_t s);
// mode 0: write |grad|^2 to out and max|grad| over the interior to hmax_bits[img];
// mode 1: write the conductivity g(|grad|^2 / k^2) to out (k from kval[img]).
void launch_cond(const float* L, size_t in_img_stride, float* out, size_t out_img_stride, Geom g, int nimg,
                 const GaussTaps& t1, int mode, int diffusivity, const float* kval, unsigned* hmax_bits,
                 cudaStream_t s);
void launch_khist(const float* g2, size_t img_stride, Geom g, int nimg, int bins, const unsigned* hmax_bits,
                  int* hist, cudaStream_t s);
void launch_kfinal(const int* hist, int bins, const unsigned* hmax_bits, int nimg, double perc, double k_override,
                   float* kval, int* fallback, cudaStream_t s);


// ---- aos.cu ----
struct Strides {  // per-image strides (floats) of the four buffers an AOS pass touches
    size_t L, c, U, out;
};
// First pass: U = column solves of (I - 2 tau A_y(c)) U = L      (strides: L, c, -, out = U)
bool launch_aos_cols(const float* L, const float* c, float* U, Strides st, Geom g, int nimg, float tau,
                     cudaStream_t s);
// Second pass: Lout = ½(U + V), V = row solves of (I - 2 tau A_x(c)) V = L   (strides: L, c, U, out)
bool launch_aos_rows(const float* L, const float* c, const float* U, float* Lout, Strides st, Geom g, int nimg,
                     float tau, cudaStream_t s);

// ---- fed.cu ----  (scheme KAZE_SCHEME_FED, A20/A21)
constexpr int kFedMaxK = 8;  // explicit steps per temporally blocked launch
struct FedTaus {
    float t[kFedMaxK];
};
// Lout = nsteps (1..kFedMaxK) explicit steps L += τ_j div(c ∇L) applied to Lin in order t[0..nsteps). Lin != Lout.
bool launch_fed_steps(const float* Lin, size_t s_in, const float* c, size_t s_c, float* Lout, size_t s_out, Geom g,
                      int nimg, const FedTaus& t, int nsteps, cudaStream_t s);

// ---- match.cu ----  
size_t match_scratch_bytes(int na, int nb);
// returns 0 or a cudaError_t / −1 (scratch too small); stats (device, optional): [matches, uncertified rows]
int match_run(const float* A, int na, const float* B, int nb, float ratio, int32_t* match, float* dist,
              void* scratch, size_t bytes, int* stats, cudaStream_t s);

// ---- hessian.cu ----  (all N levels of nimg images in one launch; level stride = plane)
// Lxy: interleaved (s·∂x L, s·∂y L) float2 planes, same element strides as the float pyramids.
void launch_hess_first(const float* Lt, float2* Lxy, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                       cudaStream_t s);
// One pass (16 B/px): Lxy and Ldet of every level of nimg images; false if some step exceeds the fused form's 32.
bool launch_hess_fused(const float* Lt, float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg,
                       const LevelTable& lt, int keep_edges, cudaStream_t s);
void launch_hess_det(const float2* Lxy, float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                     cudaStream_t s);
// Diagnostic copy of one component of an interleaved plane to/from a tightly packed w x h buffer
// (to_tight = 1: plane → tight).
void launch_component_copy(float2* plane, int comp, float* tight, int to_tight, Geom g, cudaStream_t s);

// ---- detect.cu ----
struct DetectParams {
    float threshold;
    float edge_ratio;
    int cap;
    int exact;     // exact σ window at levels i±1 (A22)
    int refine3d;  // 3-D (x, y, level) fit (A23)
};
// Candidate bitmap words per row: 30 columns per 32-bit word (bit b of word w ↔ column 30·w + b).
int nms_words(int W);
// returns the number of kernels launched (the mark pass, one or two launches, + the row count)
int launch_nms_mark(const float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt, DetectParams dp,
                    uint32_t* bitmap, int* rowcnt, cudaStream_t s);
void launch_kp_scan(const int* rowcnt, int rows_per_img, int nimg, int* rowoff, int* counts, cudaStream_t s);
void launch_kp_emit(const float* Ldet, size_t img_stride, Geom g, int nimg, const LevelTable& lt,
                    DetectParams dp, const uint32_t* bitmap, const int* rowcnt, const int* rowoff, kaze_keypoint* kps,
                    cudaStream_t s);

// ---- describe.cu ----
void init_describe_tables();
// texs: [nimg][N] texture objects over the Lxy planes (linear filtering, clamp) for the M-SURF samples.
// Keypoints whose level lies outside [lvl_lo, lvl_hi] get a zero descriptor, angle 0 and flags = 1.
// work: a device counter zeroed before the launch (dynamic keypoint distribution), or nullptr (static stride);
// overlapped: the pass shares the GPU with the next chunk's scale space (smaller persistent grid).
void launch_describe(const float2* Lxy, const cudaTextureObject_t* texs, size_t img_stride, Geom g, int nimg, int N,
                     int lvl_lo, int lvl_hi, int* work, int overlapped, kaze_keypoint* kps, const int* counts, int cap, float* desc, int nwin, int keep_angle,
                     cudaStream_t s);

__host__ __device__ inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Conductivity g(q), q = |∇|²/k² (Eq. 3): 2 = g2, 1 = g1, 3 = Weickert's 1 − exp(−3.315/q⁴) (A24;
// expm1 keeps it accurate where 3.315/q⁴ is tiny, and q⁴ → 0 gives exactly 1).
__device__ __forceinline__ float diffusivity_g(float q, int kind) {
    if (kind == 2) {
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + q));
        return r;
    }
    if (kind == 1) return __expf(-q);
    const float q2 = q * q;
    return -expm1f(-3.315f / (q2 * q2));
}

// Hides a base pointer from re-association, so `opaque(p) + (unsigned)i` compiles to ONE IMAD.WIDE.U32 per address
// instead of a 64-bit index add + LEA/LEA.HI.X pair (the compiler otherwise folds the 64-bit plane offset into
// every index).
template <class T>
__device__ __forceinline__ T* opaque(T* p) {
    asm("" : "+l"(p));
    return p;
}

}  // namespace kz
