/*
 * kazeref.h — plain, slow, fp64 CPU ORACLE for the KAZE hot path of arXiv 1706.06750.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or link anything under oracle/.
 * The product path (paper_1706_06750_b200/) never does: it shares no code, header,
 * table or constant with this file, and this file includes nothing from it.
 *
 * Citations: "P:Lnnn" = PAPER.md line nnn (section / equation in brackets);
 * "A<n>" = reading n of DESIGN.md §3 (the ambiguity register), where the paper is
 * silent, garbled or self-contradictory.
 *
 * Conventions: images are row-major H x W arrays of double (index y*W + x).
 * Every border is replicate (clamp-to-edge) [A16].  All arithmetic is fp64.
 * Functions return 0 on success and a negative value on invalid arguments.
 */
#ifndef KAZEREF_H
#define KAZEREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t octaves;        /* O  (Eq. 6)                         */
    int32_t sublevels;      /* S                                              */
    double  sigma0;         /* σ0 (Eq. 6; prefilter P:L255)                    */
    double  k_percentile;   /* percentile of the gradient histogram (A7) */
    int32_t k_bins;         /* histogram bins (A7)                            */
    int32_t diffusivity;    /* 1 = g1, 2 = g2 (Eq. 3)               */
    double  k_override;     /* > 0: use this k instead of estimating it        */
    double  threshold;      /* detector threshold (A11)            */
    double  edge_ratio;     /* r of Eq. 12; <= 0 disables the test */
    int32_t ori_windows;    /* number of sliding-window centres (A14), default 42 */
    int32_t keep_angle;     /* 1: describe with the angles already in kps (stage-isolated use) */
    int32_t scheme;         /* 0 = AOS (Eq. 4, BASELINE north_star, A1); 1 = FED cycles (Eq. 5, A20) */
    double  tau_max;        /* FED stability bound of one explicit step (A20), default 0.25 */
    int32_t exact_window;   /* 0 = approximate 3x3x3 test (A11); 1 = exact σ window at levels i±1 (A22) */
    int32_t refine3d;       /* 0 = 2-D sub-pixel fit (A13); 1 = 3-D (x, y, σ) fit */
} kazeref_params;

typedef struct {
    double  x, y;           /* sub-pixel position      */
    double  sigma;          /* σ_i of the detection level            */
    double  response;       /* Ldet at the integer extremum          */
    double  angle;          /* dominant orientation in [0, 2π)       */
    int32_t level, octave, sublevel;
    int32_t degenerate;     /* 1: all-zero orientation samples       */
} kazeref_kp;

void kazeref_default_params(kazeref_params* p);

/* Eq. 6 (reading A3) and Eq. 7; integer derivative step (A9). */
int kazeref_schedule(int O, int S, double sigma0, double* sigma, double* t, int32_t* step);

/* Sampled normalised Gaussian, radius ceil(3σ) (min 1) [A6].  taps has 2r+1 entries. */
int kazeref_gaussian_taps(double sigma, double* taps, int32_t* radius);

/* 2-D clamped convolution with the product Gaussian kernel [A6, A16]. */
int kazeref_gaussian_blur(const double* in, int W, int H, double sigma, double* out);

/* Scharr first derivative in per-pixel units, taps at 0, ±s (A8, A10):
 * dir 0: d/dx = Σ_dy w(dy)·(I(x+s, y+dy) − I(x−s, y+dy)) / (2s), w = (3,10,3)/16 at dy = −s,0,s
 * dir 1: the transpose. */
int kazeref_scharr(const double* in, int W, int H, int s, int dir, double* out);

/* Contrast factor k (reading A7).  hist may be NULL. */
int kazeref_contrast_k(const double* L0, int W, int H, double perc, int bins,
                       double* k, int64_t* hist, int32_t* fallback);

/* Conductivity c = g(|∇(G_1 * L)|) (Eqs. 2-3, reading A5); diffusivity 1 = g1, 2 = g2,
 * 3 = Weickert's g3 = 1 − exp(−3.315 / (|∇|/k)^8) (1 at |∇| = 0, reading A24). */
int kazeref_conductivity(const double* L, int W, int H, double k, int diffusivity, double* c);

/* Thomas algorithm for a_j x_{j-1} + b_j x_j + c_j x_{j+1} = d_j (a_0, c_{n-1} ignored). */
int kazeref_thomas(int n, const double* a, const double* b, const double* c, const double* d, double* x);

/* One AOS step of Eq. 4 (readings A1, A2):
 * L_new = ½[(I − 2τA_y(c))⁻¹ + (I − 2τA_x(c))⁻¹] L.   U (column solves) / V (row solves) may be NULL. */
int kazeref_aos_step(const double* L, const double* c, int W, int H, double tau,
                     double* Lnew, double* U, double* V);

/* FED step sizes of Eq. 5: τ_j = τ_max / (2 cos²(π (2j+1)/(4n+2))), j = 0..n−1. */
int kazeref_fed_taus(int n, double tau_max, double* taus);

/* One FED cycle reaching time T exactly (A20): the smallest n with τ_max·n(n+1)/3 >= T, the Eq. 5 steps scaled by
 * q = T / (τ_max·n(n+1)/3).  Writes at most cap steps; returns n (< 0 on error). */
int kazeref_fed_cycle(double T, double tau_max, double* taus, int cap);

/* Rounding-stable application order of a cycle's steps (A21).  With c fixed every step is a polynomial in the
 * same matrix A, so the cycle Π_j (I + τ_j A) does not depend on the order in exact arithmetic, but its rounding
 * does (P_m, S_m below grow like 1e12 for n = 29 in natural order).  Order: j_m = (κ·m) mod n with κ ∈ [1, n),
 * gcd(κ, n) = 1, minimising G(κ) = max_m max_μ |P_m(μ)| · max_μ |S_{m+1}(μ)|, P_m = Π_{i≤m}(1 − τ_{j_i} μ),
 * S_{m+1} = Π_{i>m}(1 − τ_{j_i} μ), μ ∈ {8i/1024 : i = 0..1024}; ties → smallest κ.  Returns κ. */
int kazeref_fed_order(const double* taus, int n, int32_t* order);

/* One explicit diffusion step (A20): L⁺(p) = L(p) + τ Σ_{q ∈ N4(p)} ½(c(p) + c(q)) (L(q) − L(p)), neighbours outside
 * the image contribute nothing (Neumann). */
int kazeref_fed_step(const double* L, const double* c, int W, int H, double tau, double* out);

/* Nonlinear scale space: L_0 = G(σ0)*I, then N−1 AOS steps (A1) or FED cycles (scheme 1, A20).
 * levels: N*H*W doubles.  k_out / fallback may be NULL. */
int kazeref_scale_space(const float* img, int W, int H, const kazeref_params* p,
                        double* levels, double* k_out, int32_t* fallback);

/* Multiscale derivatives + scale-normalised Hessian determinant (Eq. 8, A9, A10):
 * Lx = s·∂x L, Ly = s·∂y L, Ldet = s⁴(∂xx L·∂yy L − (∂yx L)²), second derivatives composed on
 * the materialised first derivatives. */
int kazeref_hessian(const double* L, int W, int H, int s, double* Lx, double* Ly, double* Ldet);

/* Edge test (Eqs. 9-12, A12) + 2-D quadratic sub-pixel fit (A13)
 * on a 3x3 response patch D (row-major, D[4] centre).  Returns 1 = keep, 0 = reject. */
int kazeref_refine(const double* D, double edge_ratio, double* dx, double* dy);

/* 3x3x3 extrema over levels 1..N-2 (A11-A13), brute-force scan.
 * Ldet: N*H*W.  Writes up to cap keypoints in (level, y, x) order; returns the true count. */
/* 3-D quadratic fit of the response in (x, y, level) from the 3x3x3 block D27[l][row][col] (l = level −1..+1)
 * with central differences (reading A23): the 2-D edge test of kazeref_refine on the centre slice first, then
 * δ = −H₃⁻¹∇D; keep iff |det H₃| >= 1e-12 and |δx|, |δy|, |δs| <= 1.  ds is in level units. */
int kazeref_refine3d(const double* D27, double edge_ratio, double* dx, double* dy, double* ds);

/* Window radius of the exact procedure at level i (reading A22): r_i = max(1, floor(s_i / 2)), s_i the
 * integer derivative step (A9) — a (2r_i+1)² window, about σ_i pixels on a side. */
int kazeref_exact_radius(int step);

/* Extrema with the detector variants of SURVEY §8 f2: exact (0/1, A22) and refine3d (0/1, A23); step[N] is the
 * per-level derivative step (used by the exact window).  kazeref_extrema = both off. */
int64_t kazeref_extrema2(const double* Ldet, int N, int W, int H, int S, const double* sigma, const int32_t* step,
                         double threshold, double edge_ratio, int exact, int refine3d, kazeref_kp* kps, int64_t cap);
int64_t kazeref_extrema(const double* Ldet, int N, int W, int H, int S, const double* sigma,
                        double threshold, double edge_ratio, kazeref_kp* kps, int64_t cap);

/* Bilinear sample with clamped taps [A14, A16]. */
double kazeref_bilinear(const double* img, int W, int H, double px, double py);

/* Dominant orientation (reading A14). */
double kazeref_orientation(const double* Lx, const double* Ly, int W, int H,
                           double x, double y, double sigma, int nwin, int32_t* degenerate);

/* 64-D M-SURF descriptor (reading A15).  Returns 1 if degenerate. */
int kazeref_descriptor(const double* Lx, const double* Ly, int W, int H,
                       double x, double y, double sigma, double angle, double* desc);

/* Full path for one image: scale space → Hessian → extrema → orientation → descriptor.
 * Optional outputs (NULL to skip): levels/Lx/Ly/Ldet (N*H*W each), desc (cap*64).
 * Returns the true keypoint count (only the first cap are written/described), < 0 on error.
 * (Stage-isolated description with given angles: kazeref_describe with keep_angle = 1.) */
int64_t kazeref_run(const float* img, int W, int H, const kazeref_params* p,
                    kazeref_kp* kps, int64_t cap, double* desc,
                    double* k_out, int32_t* fallback,
                    double* levels, double* Lx, double* Ly, double* Ldet);

/* Orientation (unless keep_angle) + descriptors for given keypoints on given Lx/Ly pyramids. */
int kazeref_describe(const double* Lx, const double* Ly, int N, int W, int H,
                     kazeref_kp* kps, int64_t n, int nwin, int keep_angle, double* desc);

/* Brute-force descriptor matching (reading A25): for every a, the nearest and
 * second-nearest b by L2 distance among the non-degenerate (nonzero) b (ties → lower index); keep iff
 * d1 < ratio·d2 (d2 = ∞ with fewer than two candidates) and the symmetric cross-check holds (a is the nearest
 * non-degenerate a of b, same tie rule).  match[a] = b or −1; dist[a] = d1 (or −1); second[a] = d2 (∞ → −1).
 * Degenerate a never match.  A: na x 64, B: nb x 64, row-major.  Returns the number of matches. */
int64_t kazeref_match(const double* A, int na, const double* B, int nb, double ratio,
                      int32_t* match, double* dist, double* second);

/* Batch of n images, OpenMP over images only (cpu_baseline timing).  counts[n]. */
int kazeref_run_batch(const float* imgs, int n, int W, int H, const kazeref_params* p,
                      int64_t cap, int nthreads, int64_t* counts);

#ifdef __cplusplus
}
#endif
#endif
