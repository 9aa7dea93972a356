/*
 * kazeref.c — plain, slow, obviously-correct fp64 CPU oracle for the KAZE hot path
 * (arXiv 1706.06750).  TEST INFRASTRUCTURE ONLY (see kazeref.h): the product CUDA path
 * never loads it, and it includes nothing from the product.
 *
 * Style: scalar loops in the paper's order and notation; 2-D clamped convolutions instead
 * of separable passes; a textbook Thomas solve per line; brute-force 26-neighbour scans.
 * No blocking, fusion or reordering.  Each function cites the passage it follows; the
 * readings A1..A26 are listed in DESIGN.md §3.
 */
#include "kazeref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KR_PI 3.14159265358979323846

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Image value with replicate border [A16]. */
static double at(const double* img, int W, int H, int x, int y) {
    return img[(size_t)clampi(y, 0, H - 1) * W + clampi(x, 0, W - 1)];
}

void kazeref_default_params(kazeref_params* p) {
    p->octaves = 4;          /* S:L118 defaults, "KAZE defaults" of BASELINE configs[1] */
    p->sublevels = 4;
    p->sigma0 = 1.6;
    p->k_percentile = 0.7;
    p->k_bins = 300;
    p->diffusivity = 2;
    p->k_override = 0.0;
    p->threshold = 1e-3;
    p->edge_ratio = 10.0;
    p->ori_windows = 42;
    p->keep_angle = 0;
    p->scheme = 0;
    p->tau_max = 0.25;
    p->exact_window = 0;
    p->refine3d = 0;
}

/* ---------------------------------------------------------------------------------------
 * Scale schedule.  Eq. 6 printed as σ0·2^{(o+s)/S}; read as σ0·2^{o + s/S} [A3]
 * (SPEC's example σ(o=1,s=0) = 3.2).  Eq. 7: t_i = σ_i²/2.  Level i = o·S + s,
 * N = O·S levels at full resolution [A4].  Derivative step of Eq. 8:
 * s_i = max(1, floor(σ_i + 1/2)) [A9].
 * ------------------------------------------------------------------------------------- */
int kazeref_schedule(int O, int S, double sigma0, double* sigma, double* t, int32_t* step) {
    if (O < 1 || S < 1 || !(sigma0 > 0)) return -1;
    for (int o = 0; o < O; ++o) {
        for (int s = 0; s < S; ++s) {
            int i = o * S + s;
            double sg = sigma0 * pow(2.0, (double)o + (double)s / (double)S);
            if (sigma) sigma[i] = sg;
            if (t) t[i] = 0.5 * sg * sg;
            if (step) {
                int st = (int)floor(sg + 0.5);
                step[i] = st < 1 ? 1 : st;
            }
        }
    }
    return 0;
}

/* Sampled Gaussian exp(−x²/(2σ²)) at integer offsets |x| <= r, r = ceil(3σ) (min 1), normalised
 * to unit sum [A6].  P:L174-175: "convolution of the image with Gaussian of standard deviation σ". */
int kazeref_gaussian_taps(double sigma, double* taps, int32_t* radius) {
    if (!(sigma > 0)) return -1;
    int r = (int)ceil(3.0 * sigma);
    if (r < 1) r = 1;
    if (radius) *radius = r;
    if (taps) {
        double sum = 0.0;
        for (int i = -r; i <= r; ++i) {
            taps[i + r] = exp(-(double)(i * i) / (2.0 * sigma * sigma));
            sum += taps[i + r];
        }
        for (int i = 0; i < 2 * r + 1; ++i) taps[i] /= sum;
    }
    return 0;
}

/* 2-D clamped convolution with the product kernel g(dx)·g(dy) — the plain definition, not the
 * separable passes (P:L255 prefilter with σ0; "two-dimensional Gaussian convolution"). */
int kazeref_gaussian_blur(const double* in, int W, int H, double sigma, double* out) {
    if (W < 1 || H < 1 || !in || !out) return -1;
    int32_t r;
    if (kazeref_gaussian_taps(sigma, NULL, &r)) return -1;
    double* g = (double*)malloc(sizeof(double) * (2 * r + 1));
    kazeref_gaussian_taps(sigma, g, &r);
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx)
                    acc += g[dy + r] * g[dx + r] * at(in, W, H, x + dx, y + dy);
            out[(size_t)y * W + x] = acc;
        }
    }
    free(g);
    return 0;
}

/* Scharr first derivative at step s in per-pixel units [A8, A10]: the 3x3 Scharr kernel dilated
 * to taps at {−s, 0, +s} ("Concatenated Scharr filter of step size ...").
 * Derivative taps (−1, 0, +1)/(2s); cross-axis smoothing taps (3, 10, 3)/16. */
int kazeref_scharr(const double* in, int W, int H, int s, int dir, double* out) {
    if (W < 1 || H < 1 || s < 1 || !in || !out || (dir != 0 && dir != 1)) return -1;
    static const double w[3] = {3.0 / 16.0, 10.0 / 16.0, 3.0 / 16.0};
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int k = -1; k <= 1; ++k) {
                if (dir == 0)
                    acc += w[k + 1] * (at(in, W, H, x + s, y + k * s) - at(in, W, H, x - s, y + k * s));
                else
                    acc += w[k + 1] * (at(in, W, H, x + k * s, y + s) - at(in, W, H, x + k * s, y - s));
            }
            out[(size_t)y * W + x] = acc / (2.0 * s);
        }
    }
    return 0;
}

/* Contrast factor k: "image gradient histogram is computed to obtain the contrast parameter k in
 * an automatic procedure" (k of Eq. 3).  Reading A7:
 *   Ls = G(1) * L0;  gx, gy = Scharr step 1 of Ls;  g = sqrt(gx² + gy²) over the interior
 *   [1, W−2] x [1, H−2];  hmax = max g;  histogram of the n values with g > 0 into `bins` bins,
 *   bin = min(floor(bins·g/hmax), bins−1);  thr = floor(perc·n);  b = first bin whose cumulative
 *   count >= thr;  k = hmax·(b+1)/bins.   n == 0 → k = 0.03, fallback = 1. */
int kazeref_contrast_k(const double* L0, int W, int H, double perc, int bins,
                       double* k, int64_t* hist, int32_t* fallback) {
    if (W < 3 || H < 3 || bins < 1 || !(perc > 0 && perc < 1) || !k) return -1;
    size_t np = (size_t)W * H;
    double* Ls = (double*)malloc(sizeof(double) * np);
    double* gx = (double*)malloc(sizeof(double) * np);
    double* gy = (double*)malloc(sizeof(double) * np);
    int64_t* h = (int64_t*)calloc((size_t)bins, sizeof(int64_t));
    kazeref_gaussian_blur(L0, W, H, 1.0, Ls);
    kazeref_scharr(Ls, W, H, 1, 0, gx);
    kazeref_scharr(Ls, W, H, 1, 1, gy);
    double hmax = 0.0;
    for (int y = 1; y < H - 1; ++y)
        for (int x = 1; x < W - 1; ++x) {
            size_t i = (size_t)y * W + x;
            double g = sqrt(gx[i] * gx[i] + gy[i] * gy[i]);
            if (g > hmax) hmax = g;
        }
    int64_t n = 0;
    for (int y = 1; y < H - 1; ++y)
        for (int x = 1; x < W - 1; ++x) {
            size_t i = (size_t)y * W + x;
            double g = sqrt(gx[i] * gx[i] + gy[i] * gy[i]);
            if (g > 0.0) {
                int b = (int)floor((double)bins * g / hmax);
                if (b > bins - 1) b = bins - 1;
                h[b] += 1;
                n += 1;
            }
        }
    if (n == 0) {
        *k = 0.03;
        if (fallback) *fallback = 1;
    } else {
        int64_t thr = (int64_t)floor(perc * (double)n);
        int64_t cum = 0;
        int b = 0;
        for (b = 0; b < bins; ++b) {
            cum += h[b];
            if (cum >= thr) break;
        }
        if (b >= bins) b = bins - 1;
        *k = hmax * (double)(b + 1) / (double)bins;
        if (fallback) *fallback = 0;
    }
    if (hist) memcpy(hist, h, sizeof(int64_t) * (size_t)bins);
    free(Ls); free(gx); free(gy); free(h);
    return 0;
}

/* Perona–Malik conductivity c = g(|∇I_σ|) (Eq. 2) with g1 / g2 of Eq. 3
 * (P:L124-126); ∇I_σ = Scharr step 1 of G(σ=1) * L (reading A5; "L_smooth ... first order
 * ... derivatives ... Scharr"). */
int kazeref_conductivity(const double* L, int W, int H, double k, int diffusivity, double* c) {
    if (!(k > 0) || diffusivity < 1 || diffusivity > 3) return -1;
    size_t np = (size_t)W * H;
    double* Ls = (double*)malloc(sizeof(double) * np);
    double* gx = (double*)malloc(sizeof(double) * np);
    double* gy = (double*)malloc(sizeof(double) * np);
    kazeref_gaussian_blur(L, W, H, 1.0, Ls);
    kazeref_scharr(Ls, W, H, 1, 0, gx);
    kazeref_scharr(Ls, W, H, 1, 1, gy);
    for (size_t i = 0; i < np; ++i) {
        double q = (gx[i] * gx[i] + gy[i] * gy[i]) / (k * k);
        if (diffusivity == 2) c[i] = 1.0 / (1.0 + q);
        else if (diffusivity == 1) c[i] = exp(-q);
        else c[i] = q > 0.0 ? 1.0 - exp(-3.315 / (q * q * q * q)) : 1.0;  /* (|∇|/k)^8 = q^4 (A24) */
    }
    free(Ls); free(gx); free(gy);
    return 0;
}

/* Textbook Thomas algorithm (no pivoting; the AOS matrices are strictly diagonally dominant [A2]). */
int kazeref_thomas(int n, const double* a, const double* b, const double* c, const double* d, double* x) {
    if (n < 1) return -1;
    double* cp = (double*)malloc(sizeof(double) * n);
    double* dp = (double*)malloc(sizeof(double) * n);
    cp[0] = (n > 1 ? c[0] : 0.0) / b[0];
    dp[0] = d[0] / b[0];
    for (int j = 1; j < n; ++j) {
        double m = b[j] - a[j] * cp[j - 1];
        cp[j] = (j < n - 1 ? c[j] : 0.0) / m;
        dp[j] = (d[j] - a[j] * dp[j - 1]) / m;
    }
    x[n - 1] = dp[n - 1];
    for (int j = n - 2; j >= 0; --j) x[j] = dp[j] - cp[j] * x[j + 1];
    free(cp); free(dp);
    return 0;
}

/* Solve (I − 2τA(c)) x = d for one line of n samples with stride `stride` [A2]:
 * (A)_{j,j±1} = (c_j + c_{j±1})/2, (A)_{jj} = −Σ off-diagonals (Neumann: the end samples have one
 * neighbour).  Hence off-diagonals −τ(c_j + c_{j+1}) and diagonal 1 + τ(q_{j−1} + q_j). */
static void aos_line(const double* Lline, const double* cline, int n, size_t stride, double tau,
                     double* out) {
    if (n < 1) return;
    double* a = (double*)malloc(sizeof(double) * n);
    double* b = (double*)malloc(sizeof(double) * n);
    double* cc = (double*)malloc(sizeof(double) * n);
    double* d = (double*)malloc(sizeof(double) * n);
    double* x = (double*)malloc(sizeof(double) * n);
    for (int j = 0; j < n; ++j) {
        double qm = (j > 0) ? cline[(size_t)j * stride] + cline[(size_t)(j - 1) * stride] : 0.0;
        double qp = (j < n - 1) ? cline[(size_t)j * stride] + cline[(size_t)(j + 1) * stride] : 0.0;
        a[j] = -tau * qm;
        cc[j] = -tau * qp;
        b[j] = 1.0 + tau * (qm + qp);
        d[j] = Lline[(size_t)j * stride];
    }
    kazeref_thomas(n, a, b, cc, d, x);
    for (int j = 0; j < n; ++j) out[(size_t)j * stride] = x[j];
    free(a); free(b); free(cc); free(d); free(x);
}

/* AOS step for Eq. 4 with m = 2 dimensions (reading A1, BASELINE north_star):
 * L_new = ½ Σ_l (I − 2τ A_l(c))⁻¹ L.   U = column systems (y direction), V = row systems (x). */
int kazeref_aos_step(const double* L, const double* c, int W, int H, double tau,
                     double* Lnew, double* U, double* V) {
    if (W < 1 || H < 1 || !(tau >= 0) || !L || !c || !Lnew) return -1;
    size_t np = (size_t)W * H;
    double* u = U ? U : (double*)malloc(sizeof(double) * np);
    double* v = V ? V : (double*)malloc(sizeof(double) * np);
    for (int x = 0; x < W; ++x) aos_line(L + x, c + x, H, (size_t)W, tau, u + x);
    for (int y = 0; y < H; ++y) aos_line(L + (size_t)y * W, c + (size_t)y * W, W, 1, tau, v + (size_t)y * W);
    for (size_t i = 0; i < np; ++i) Lnew[i] = 0.5 * (u[i] + v[i]);
    if (!U) free(u);
    if (!V) free(v);
    return 0;
}

/* FED (Eq. 5; reading A20): "perform M cycles of n explicit diffusion steps with varying step sizes". */
int kazeref_fed_taus(int n, double tau_max, double* taus) {
    if (n < 1 || !(tau_max > 0) || !taus) return -1;
    for (int j = 0; j < n; ++j) {
        double cj = cos(KR_PI * (double)(2 * j + 1) / (double)(4 * n + 2));
        taus[j] = tau_max / (2.0 * cj * cj);
    }
    return 0;
}

/* A20: n = smallest integer with τ_max·n(n+1)/3 >= T (the closed-form sum of Eq. 5's steps), i.e.
 * n = ceil(−1/2 + 1/2·sqrt(1 + 12 T / τ_max)); the steps are scaled by q = T / (τ_max·n(n+1)/3). */
int kazeref_fed_cycle(double T, double tau_max, double* taus, int cap) {
    if (!(T > 0) || !(tau_max > 0)) return -1;
    int n = (int)ceil(-0.5 + 0.5 * sqrt(1.0 + 12.0 * T / tau_max) - 1e-12);
    if (n < 1) n = 1;
    while (tau_max * n * (n + 1) / 3.0 < T) ++n;  /* guard the ceiling against rounding */
    if (taus) {
        double* t = (double*)malloc(sizeof(double) * n);
        kazeref_fed_taus(n, tau_max, t);
        double q = T / (tau_max * n * (n + 1) / 3.0);
        for (int j = 0; j < n && j < cap; ++j) taus[j] = q * t[j];
        free(t);
    }
    return n;
}

static int kr_gcd(int a, int b) { while (b) { int t = a % b; a = b; b = t; } return a; }

/* A21: choose κ by brute force over every admissible κ and every μ of the grid. */
int kazeref_fed_order(const double* taus, int n, int32_t* order) {
    if (n < 1 || !taus || !order) return -1;
    enum { NMU = 1025 };
    int best_k = 1;
    double best_g = -1.0;
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * n);
    double* pre = (double*)malloc(sizeof(double) * n);  /* max_μ |P_m| */
    double* suf = (double*)malloc(sizeof(double) * (n + 1));  /* max_μ |S_m| (S_n = 1) */
    for (int k = 1; k < (n > 1 ? n : 2); ++k) {
        if (kr_gcd(k, n) != 1) continue;
        for (int m = 0; m < n; ++m) ord[m] = (int32_t)(((long)k * m) % n);
        for (int m = 0; m < n; ++m) pre[m] = 0.0;
        for (int m = 0; m <= n; ++m) suf[m] = (m == n) ? 1.0 : 0.0;
        for (int i = 0; i < NMU; ++i) {
            double mu = 8.0 * i / (NMU - 1);
            double p = 1.0;
            for (int m = 0; m < n; ++m) {
                p *= 1.0 - taus[ord[m]] * mu;
                if (fabs(p) > pre[m]) pre[m] = fabs(p);
            }
            double s = 1.0;
            for (int m = n - 1; m >= 0; --m) {
                s *= 1.0 - taus[ord[m]] * mu;
                if (fabs(s) > suf[m]) suf[m] = fabs(s);
            }
        }
        double g = 0.0;
        for (int m = 0; m < n; ++m) {
            double v = pre[m] * suf[m + 1];
            if (v > g) g = v;
        }
        if (best_g < 0 || g < best_g) { best_g = g; best_k = k; }
    }
    for (int m = 0; m < n; ++m) order[m] = (int32_t)(((long)best_k * m) % n);
    free(ord); free(pre); free(suf);
    return best_k;
}

/* One explicit step of Eq. 1 with the conductivities held fixed (A20): the flux through the face
 * between p and its 4-neighbour q is ½(c_p + c_q)(L_q − L_p); faces on the image border carry no flux (Neumann). */
int kazeref_fed_step(const double* L, const double* c, int W, int H, double tau, double* out) {
    if (!L || !c || !out || W < 1 || H < 1) return -1;
    static const int dx[4] = {1, -1, 0, 0}, dy[4] = {0, 0, 1, -1};
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t p = (size_t)y * W + x;
            double flux = 0.0;
            for (int k = 0; k < 4; ++k) {
                int qx = x + dx[k], qy = y + dy[k];
                if (qx < 0 || qx >= W || qy < 0 || qy >= H) continue;
                size_t q = (size_t)qy * W + qx;
                flux += 0.5 * (c[p] + c[q]) * (L[q] - L[p]);
            }
            out[p] = L[p] + tau * flux;
        }
    return 0;
}

/* Nonlinear scale space (P:L255-260 with the AOS solver of Eq. 4 [A1], or the FED cycles of Eq. 5 [A20]):
 *   L_0 = G(σ0) * I  (t_0 = σ0²/2);   k from L_0 (A7) unless overridden;
 *   for i = 1..N−1:  c_i = g(|∇ G(1)*L_{i−1}|),  τ_i = t_i − t_{i−1},  L_i = AOS(L_{i−1}, c_i, τ_i)  or
 *                    L_i = FED cycle of total time τ_i applied to L_{i−1} with c_i fixed, steps in the A21 order. */
int kazeref_scale_space(const float* img, int W, int H, const kazeref_params* p,
                        double* levels, double* k_out, int32_t* fallback) {
    if (!img || !p || !levels || W < 3 || H < 3) return -1;
    int N = p->octaves * p->sublevels;
    if (N < 1) return -1;
    double* t = (double*)malloc(sizeof(double) * N);
    if (kazeref_schedule(p->octaves, p->sublevels, p->sigma0, NULL, t, NULL)) { free(t); return -1; }
    size_t np = (size_t)W * H;
    double* I = (double*)malloc(sizeof(double) * np);
    for (size_t i = 0; i < np; ++i) I[i] = (double)img[i];
    kazeref_gaussian_blur(I, W, H, p->sigma0, levels);
    double k;
    int32_t fb = 0;
    if (p->k_override > 0) {
        k = p->k_override;
    } else if (kazeref_contrast_k(levels, W, H, p->k_percentile, p->k_bins, &k, NULL, &fb)) {
        free(t); free(I); return -1;
    }
    if (k_out) *k_out = k;
    if (fallback) *fallback = fb;
    double* c = (double*)malloc(sizeof(double) * np);
    double* tmp = p->scheme == 1 ? (double*)malloc(sizeof(double) * np) : NULL;
    for (int i = 1; i < N; ++i) {
        const double* prev = levels + (size_t)(i - 1) * np;
        double* cur = levels + (size_t)i * np;
        kazeref_conductivity(prev, W, H, k, p->diffusivity, c);
        if (p->scheme == 1) {  /* FED cycle from t_{i-1} to t_i with c held fixed (A20) */
            int n = kazeref_fed_cycle(t[i] - t[i - 1], p->tau_max, NULL, 0);
            double* taus = (double*)malloc(sizeof(double) * n);
            int32_t* order = (int32_t*)malloc(sizeof(int32_t) * n);
            kazeref_fed_cycle(t[i] - t[i - 1], p->tau_max, taus, n);
            kazeref_fed_order(taus, n, order);  /* A21 */
            memcpy(cur, prev, sizeof(double) * np);
            for (int j = 0; j < n; ++j) {
                kazeref_fed_step(cur, c, W, H, taus[order[j]], tmp);
                memcpy(cur, tmp, sizeof(double) * np);
            }
            free(taus); free(order);
        } else {
            kazeref_aos_step(prev, c, W, H, t[i] - t[i - 1], cur, NULL, NULL);
        }
    }
    free(c); free(I); free(t);
    if (tmp) free(tmp);
    return 0;
}

/* Eq. 8 with readings A9/A10: first derivatives of L_i with the Scharr filter of
 * step s; second derivatives by composing a second Scharr pass on the MATERIALISED first
 * derivative (clamped reads of Lx, Ly); Lxx = ∂x(Lx), Lyy = ∂y(Ly), Lxy = ∂y(Lx).
 * Normalisation: one factor s per derivative order, so Ldet = s⁴(LxxLyy − Lxy²). */
int kazeref_hessian(const double* L, int W, int H, int s, double* Lx, double* Ly, double* Ldet) {
    if (!L || s < 1 || W < 1 || H < 1) return -1;
    size_t np = (size_t)W * H;
    double* dx = (double*)malloc(sizeof(double) * np);
    double* dy = (double*)malloc(sizeof(double) * np);
    double* dxx = (double*)malloc(sizeof(double) * np);
    double* dyy = (double*)malloc(sizeof(double) * np);
    double* dxy = (double*)malloc(sizeof(double) * np);
    kazeref_scharr(L, W, H, s, 0, dx);
    kazeref_scharr(L, W, H, s, 1, dy);
    kazeref_scharr(dx, W, H, s, 0, dxx);
    kazeref_scharr(dy, W, H, s, 1, dyy);
    kazeref_scharr(dx, W, H, s, 1, dxy);
    double s2 = (double)s * (double)s;
    for (size_t i = 0; i < np; ++i) {
        if (Lx) Lx[i] = s * dx[i];
        if (Ly) Ly[i] = s * dy[i];
        if (Ldet) Ldet[i] = s2 * s2 * (dxx[i] * dyy[i] - dxy[i] * dxy[i]);
    }
    free(dx); free(dy); free(dxx); free(dyy); free(dxy);
    return 0;
}

/* Edge elimination: Hessian of the response surface D from its 3x3 neighbourhood
 * ("calculated by 8 points around those points"), Tr = Dxx + Dyy (Eq. 10's "D_xy" read as the
 * typo it is [A12]), Det = Dxx·Dyy − Dxy² (Eq. 11); keep iff Det > 0 and Tr²/Det < (r+1)²/r
 * (Eq. 12).  Then the 2-D quadratic fit of the 3x3 response [A13]:
 * δ = −H⁻¹∇D with central differences; reject if |det H| < 1e-12 or |δx| > 1 or |δy| > 1. */
int kazeref_refine(const double* D, double edge_ratio, double* dx, double* dy) {
    /* D[(row)*3 + col], row = y+1, col = x+1 */
    double c = D[4];
    double Dxx = D[5] + D[3] - 2.0 * c;
    double Dyy = D[7] + D[1] - 2.0 * c;
    double Dxy = 0.25 * (D[8] + D[0] - D[2] - D[6]);
    double Dx = 0.5 * (D[5] - D[3]);
    double Dy = 0.5 * (D[7] - D[1]);
    double det = Dxx * Dyy - Dxy * Dxy;
    if (edge_ratio > 0) {
        double tr = Dxx + Dyy;
        if (!(det > 0.0)) return 0;
        if (!(tr * tr / det < (edge_ratio + 1.0) * (edge_ratio + 1.0) / edge_ratio)) return 0;
    }
    if (fabs(det) < 1e-12) return 0;
    double ox = -(Dyy * Dx - Dxy * Dy) / det;
    double oy = -(Dxx * Dy - Dxy * Dx) / det;
    if (fabs(ox) > 1.0 || fabs(oy) > 1.0) return 0;
    if (dx) *dx = ox;
    if (dy) *dy = oy;
    return 1;
}

int kazeref_refine3d(const double* D27, double edge_ratio, double* dx, double* dy, double* ds) {
    const double* Dm = D27;       /* level i-1 */
    const double* D = D27 + 9;    /* level i   */
    const double* Dp = D27 + 18;  /* level i+1 */
    double c = D[4];
    double Dxx = D[5] + D[3] - 2.0 * c;
    double Dyy = D[7] + D[1] - 2.0 * c;
    double Dss = Dp[4] + Dm[4] - 2.0 * c;
    double Dxy = 0.25 * (D[8] + D[0] - D[2] - D[6]);
    double Dxs = 0.25 * (Dp[5] - Dp[3] - Dm[5] + Dm[3]);
    double Dys = 0.25 * (Dp[7] - Dp[1] - Dm[7] + Dm[1]);
    double gx = 0.5 * (D[5] - D[3]), gy = 0.5 * (D[7] - D[1]), gs = 0.5 * (Dp[4] - Dm[4]);
    if (edge_ratio > 0) {  /* the 2-D edge test of Eqs. 9-12 on the detection level (A12) */
        double det2 = Dxx * Dyy - Dxy * Dxy, tr = Dxx + Dyy;
        if (!(det2 > 0.0)) return 0;
        if (!(tr * tr / det2 < (edge_ratio + 1.0) * (edge_ratio + 1.0) / edge_ratio)) return 0;
    }
    /* H = [[Dxx Dxy Dxs] [Dxy Dyy Dys] [Dxs Dys Dss]]; δ = −H⁻¹ g by the adjugate (H symmetric) */
    double A00 = Dyy * Dss - Dys * Dys, A01 = Dxs * Dys - Dxy * Dss, A02 = Dxy * Dys - Dxs * Dyy;
    double A11 = Dxx * Dss - Dxs * Dxs, A12 = Dxy * Dxs - Dxx * Dys, A22 = Dxx * Dyy - Dxy * Dxy;
    double det = Dxx * A00 + Dxy * A01 + Dxs * A02;
    if (fabs(det) < 1e-12) return 0;
    double ox = -(A00 * gx + A01 * gy + A02 * gs) / det;
    double oy = -(A01 * gx + A11 * gy + A12 * gs) / det;
    double os = -(A02 * gx + A12 * gy + A22 * gs) / det;
    if (fabs(ox) > 1.0 || fabs(oy) > 1.0 || fabs(os) > 1.0) return 0;
    if (dx) *dx = ox;
    if (dy) *dy = oy;
    if (ds) *ds = os;
    return 1;
}

int kazeref_exact_radius(int step) { return step / 2 > 1 ? step / 2 : 1; }

/* Scale-space extrema [A11]: for levels i = 1..N−2 and pixels at least 1 from the border, keep
 * (x, y) iff Ldet_i(x,y) > threshold and it is strictly greater than
 *   approximate (exact = 0): all 26 neighbours in the 3x3 windows of levels i−1, i, i+1;
 *   exact (exact = 1, A22): its 8 neighbours at level i and every in-image pixel of the
 *     (2r_i+1)² window centred on it at levels i−1 and i+1;
 * then the edge test and the 2-D fit (kazeref_refine, A13) or the 3-D fit (kazeref_refine3d, A23; σ becomes
 * σ_i·2^{δs/S}, one level being 1/S octave). */
int64_t kazeref_extrema2(const double* Ldet, int N, int W, int H, int S, const double* sigma, const int32_t* step,
                         double threshold, double edge_ratio, int exact, int refine3d, kazeref_kp* kps, int64_t cap) {
    size_t np = (size_t)W * H;
    int64_t count = 0;
    if (exact && !step) return -1;
    for (int i = 1; i < N - 1; ++i) {
        const double* D = Ldet + (size_t)i * np;
        const int r = exact ? kazeref_exact_radius(step[i]) : 1;
        for (int y = 1; y < H - 1; ++y) {
            for (int x = 1; x < W - 1; ++x) {
                double v = D[(size_t)y * W + x];
                if (!(v > threshold)) continue;
                int ismax = 1;
                for (int l = -1; l <= 1 && ismax; ++l) {
                    const double* Dl = Ldet + (size_t)(i + l) * np;
                    const int rr = l == 0 ? 1 : r;
                    for (int yy = -rr; yy <= rr && ismax; ++yy)
                        for (int xx = -rr; xx <= rr; ++xx) {
                            if (l == 0 && yy == 0 && xx == 0) continue;
                            int qx = x + xx, qy = y + yy;
                            if (qx < 0 || qx >= W || qy < 0 || qy >= H) continue;  /* in-image pixels only */
                            if (!(v > Dl[(size_t)qy * W + qx])) { ismax = 0; break; }
                        }
                }
                if (!ismax) continue;
                double ox, oy, os = 0.0;
                if (refine3d) {
                    double blk[27];
                    for (int l = -1; l <= 1; ++l)
                        for (int yy = -1; yy <= 1; ++yy)
                            for (int xx = -1; xx <= 1; ++xx)
                                blk[(l + 1) * 9 + (yy + 1) * 3 + (xx + 1)] =
                                    Ldet[(size_t)(i + l) * np + (size_t)(y + yy) * W + (x + xx)];
                    if (!kazeref_refine3d(blk, edge_ratio, &ox, &oy, &os)) continue;
                } else {
                    double patch[9];
                    for (int yy = -1; yy <= 1; ++yy)
                        for (int xx = -1; xx <= 1; ++xx)
                            patch[(yy + 1) * 3 + (xx + 1)] = D[(size_t)(y + yy) * W + (x + xx)];
                    if (!kazeref_refine(patch, edge_ratio, &ox, &oy)) continue;
                }
                if (kps && count < cap) {
                    kazeref_kp* k = &kps[count];
                    k->x = x + ox;
                    k->y = y + oy;
                    k->sigma = refine3d ? sigma[i] * pow(2.0, os / S) : sigma[i];
                    k->response = v;
                    k->angle = 0.0;
                    k->level = i;
                    k->octave = i / S;
                    k->sublevel = i % S;
                    k->degenerate = 0;
                }
                count += 1;
            }
        }
    }
    return count;
}

int64_t kazeref_extrema(const double* Ldet, int N, int W, int H, int S, const double* sigma,
                        double threshold, double edge_ratio, kazeref_kp* kps, int64_t cap) {
    return kazeref_extrema2(Ldet, N, W, H, S, sigma, NULL, threshold, edge_ratio, 0, 0, kps, cap);
}

/* Bilinear interpolation with clamped taps (reading A14: bilinear reads; A16 replicate). */
double kazeref_bilinear(const double* img, int W, int H, double px, double py) {
    double fx0 = floor(px), fy0 = floor(py);
    int x0 = (int)fx0, y0 = (int)fy0;
    double fx = px - fx0, fy = py - fy0;
    double v00 = at(img, W, H, x0, y0), v10 = at(img, W, H, x0 + 1, y0);
    double v01 = at(img, W, H, x0, y0 + 1), v11 = at(img, W, H, x0 + 1, y0 + 1);
    return (1.0 - fy) * ((1.0 - fx) * v00 + fx * v10) + fy * ((1.0 - fx) * v01 + fx * v11);
}

/* Map an angle difference to (−π, π]. */
static double wrap_pi(double a) {
    while (a > KR_PI) a -= 2.0 * KR_PI;
    while (a <= -KR_PI) a += 2.0 * KR_PI;
    return a;
}

/* Dominant orientation [A14]: samples at kp + σ(u, v) for integers
 * u² + v² <= 36 ("sampling step of size σ_i in a circular area of radius 6σ_i"), each the
 * bilinear (Lx, Ly) weighted by a Gaussian of std 2.5σ_i, i.e. exp(−(u²+v²)/12.5); the weighted
 * responses are points in vector space; for nwin window centres θ_k = 2πk/nwin sum the points whose
 * angle lies strictly within ±π/6 of θ_k ("sliding circle segment covering an angle of π/3");
 * the orientation is the angle of the longest summed vector (first k on ties), in [0, 2π). */
double kazeref_orientation(const double* Lx, const double* Ly, int W, int H,
                           double x, double y, double sigma, int nwin, int32_t* degenerate) {
    double rx[113], ry[113], ph[113];
    int ns = 0;
    for (int v = -6; v <= 6; ++v)
        for (int u = -6; u <= 6; ++u) {
            if (u * u + v * v > 36) continue;
            double px = x + sigma * u, py = y + sigma * v;
            double w = exp(-(double)(u * u + v * v) / 12.5);
            rx[ns] = w * kazeref_bilinear(Lx, W, H, px, py);
            ry[ns] = w * kazeref_bilinear(Ly, W, H, px, py);
            double a = atan2(ry[ns], rx[ns]);
            if (a < 0) a += 2.0 * KR_PI;
            ph[ns] = a;
            ns += 1;
        }
    double best = 0.0, bx = 0.0, by = 0.0;
    for (int k = 0; k < nwin; ++k) {
        double th = 2.0 * KR_PI * (double)k / (double)nwin;
        double sx = 0.0, sy = 0.0;
        for (int j = 0; j < ns; ++j) {
            if (fabs(wrap_pi(ph[j] - th)) < KR_PI / 6.0) {
                sx += rx[j];
                sy += ry[j];
            }
        }
        double m = sx * sx + sy * sy;
        if (m > best) { best = m; bx = sx; by = sy; }
    }
    if (!(best > 0.0)) {
        if (degenerate) *degenerate = 1;
        return 0.0;
    }
    if (degenerate) *degenerate = 0;
    double ang = atan2(by, bx);
    if (ang < 0) ang += 2.0 * KR_PI;
    if (ang >= 2.0 * KR_PI) ang -= 2.0 * KR_PI;
    return ang;
}

/* 64-D M-SURF descriptor [A15]:
 * a 24x24 grid of samples at step σ_i (the 24σ_i x 24σ_i window), symmetric about the keypoint
 * (u, v ∈ {−11.5, …, 11.5}), rotated by the dominant orientation θ; (Lx, Ly) bilinear at each
 * sample, expressed in the rotated frame (du, dv) ("derivatives according to the dominant
 * orientation"); 4x4 subregions of 9x9 samples starting every 5 samples (9σ_i, overlapping);
 * per subregion Σ w1·du, Σ w1·dv, Σ|w1·du|, Σ|w1·dv| with w1 a Gaussian of std 2.5 (σ_i units)
 * about the subregion centre (5a − 7.5, 5b − 7.5); each subregion vector weighted by a 4x4
 * Gaussian mask of std 1.5 (subregion-index units) about the keypoint; concatenated to 64 values
 * (index 4(4b + a) + j) and normalised to unit length (zero vector if degenerate). */
int kazeref_descriptor(const double* Lx, const double* Ly, int W, int H,
                       double x, double y, double sigma, double angle, double* desc) {
    double co = cos(angle), si = sin(angle);
    double du[24][24], dv[24][24];  /* [p][q], p along u, q along v */
    for (int p = 0; p < 24; ++p)
        for (int q = 0; q < 24; ++q) {
            double u = p - 11.5, v = q - 11.5;
            double px = x + sigma * (u * co - v * si);
            double py = y + sigma * (u * si + v * co);
            double gx = kazeref_bilinear(Lx, W, H, px, py);
            double gy = kazeref_bilinear(Ly, W, H, px, py);
            du[p][q] = gx * co + gy * si;
            dv[p][q] = -gx * si + gy * co;
        }
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
            double cu = 5.0 * a - 7.5, cv = 5.0 * b - 7.5;
            double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
            for (int p = 5 * a; p <= 5 * a + 8; ++p)
                for (int q = 5 * b; q <= 5 * b + 8; ++q) {
                    double u = p - 11.5, v = q - 11.5;
                    double w1 = exp(-((u - cu) * (u - cu) + (v - cv) * (v - cv)) / (2.0 * 2.5 * 2.5));
                    s0 += w1 * du[p][q];
                    s1 += w1 * dv[p][q];
                    s2 += fabs(w1 * du[p][q]);
                    s3 += fabs(w1 * dv[p][q]);
                }
            double w2 = exp(-((a - 1.5) * (a - 1.5) + (b - 1.5) * (b - 1.5)) / (2.0 * 1.5 * 1.5));
            int base = 4 * (4 * b + a);
            desc[base + 0] = w2 * s0;
            desc[base + 1] = w2 * s1;
            desc[base + 2] = w2 * s2;
            desc[base + 3] = w2 * s3;
        }
    double n2 = 0.0;
    for (int i = 0; i < 64; ++i) n2 += desc[i] * desc[i];
    if (!(n2 > 0.0)) {
        for (int i = 0; i < 64; ++i) desc[i] = 0.0;
        return 1;
    }
    double inv = 1.0 / sqrt(n2);
    for (int i = 0; i < 64; ++i) desc[i] *= inv;
    return 0;
}

int kazeref_describe(const double* Lx, const double* Ly, int N, int W, int H,
                     kazeref_kp* kps, int64_t n, int nwin, int keep_angle, double* desc) {
    size_t np = (size_t)W * H;
    for (int64_t j = 0; j < n; ++j) {
        kazeref_kp* k = &kps[j];
        if (k->level < 0 || k->level >= N) return -1;
        const double* lx = Lx + (size_t)k->level * np;
        const double* ly = Ly + (size_t)k->level * np;
        if (!keep_angle) {
            int32_t deg = 0;
            k->angle = kazeref_orientation(lx, ly, W, H, k->x, k->y, k->sigma, nwin, &deg);
            k->degenerate = deg;
        }
        if (desc) kazeref_descriptor(lx, ly, W, H, k->x, k->y, k->sigma, k->angle, desc + j * 64);
    }
    return 0;
}

int64_t kazeref_run(const float* img, int W, int H, const kazeref_params* p,
                    kazeref_kp* kps, int64_t cap, double* desc,
                    double* k_out, int32_t* fallback,
                    double* levels, double* Lx, double* Ly, double* Ldet) {
    if (!img || !p || W < 3 || H < 3) return -1;
    int N = p->octaves * p->sublevels;
    if (N < 1) return -1;
    size_t np = (size_t)W * H;
    double* sg = (double*)malloc(sizeof(double) * N);
    int32_t* st = (int32_t*)malloc(sizeof(int32_t) * N);
    kazeref_schedule(p->octaves, p->sublevels, p->sigma0, sg, NULL, st);
    double* lv = levels ? levels : (double*)malloc(sizeof(double) * np * N);
    double* lx = Lx ? Lx : (double*)malloc(sizeof(double) * np * N);
    double* ly = Ly ? Ly : (double*)malloc(sizeof(double) * np * N);
    double* ld = Ldet ? Ldet : (double*)malloc(sizeof(double) * np * N);
    int64_t count = -1;
    if (kazeref_scale_space(img, W, H, p, lv, k_out, fallback) == 0) {
        for (int i = 0; i < N; ++i)
            kazeref_hessian(lv + (size_t)i * np, W, H, st[i], lx + (size_t)i * np,
                            ly + (size_t)i * np, ld + (size_t)i * np);
        count = kazeref_extrema2(ld, N, W, H, p->sublevels, sg, st, p->threshold, p->edge_ratio, p->exact_window,
                                 p->refine3d, kps, cap);
        int64_t nd = count < cap ? count : cap;
        if (kps && nd > 0) kazeref_describe(lx, ly, N, W, H, kps, nd, p->ori_windows, 0, desc);
    }
    if (!levels) free(lv);
    if (!Lx) free(lx);
    if (!Ly) free(ly);
    if (!Ldet) free(ld);
    free(sg); free(st);
    return count;
}

/* A25: the matcher S:L399-440 defines (the paper cites matching as the application, but defines no
 * matcher).  Distances are computed from the descriptor difference, in fp64, in the plain double loop. */
static double kr_dist(const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < 64; ++i) {
        double d = a[i] - b[i];
        s += d * d;
    }
    return sqrt(s);
}

static int kr_degenerate(const double* a) {
    for (int i = 0; i < 64; ++i)
        if (a[i] != 0.0) return 0;
    return 1;
}

/* nearest (and second) non-degenerate row of Y for x; ties → lower index. */
static void kr_nearest(const double* x, const double* Y, int ny, const int* ydeg, int* i1, double* d1, double* d2) {
    *i1 = -1;
    *d1 = INFINITY;
    *d2 = INFINITY;
    for (int j = 0; j < ny; ++j) {
        if (ydeg[j]) continue;
        double d = kr_dist(x, Y + (size_t)j * 64);
        if (d < *d1) {
            *d2 = *d1;
            *d1 = d;
            *i1 = j;
        } else if (d < *d2) {
            *d2 = d;
        }
    }
}

int64_t kazeref_match(const double* A, int na, const double* B, int nb, double ratio,
                      int32_t* match, double* dist, double* second) {
    if (na < 0 || nb < 0 || !(ratio > 0 && ratio <= 1) || (na > 0 && (!A || !match)) || (nb > 0 && !B)) return -1;
    int* adeg = (int*)malloc(sizeof(int) * (na > 0 ? na : 1));
    int* bdeg = (int*)malloc(sizeof(int) * (nb > 0 ? nb : 1));
    for (int i = 0; i < na; ++i) adeg[i] = kr_degenerate(A + (size_t)i * 64);
    for (int j = 0; j < nb; ++j) bdeg[j] = kr_degenerate(B + (size_t)j * 64);
    int64_t count = 0;
    for (int i = 0; i < na; ++i) {
        match[i] = -1;
        if (dist) dist[i] = -1.0;
        if (second) second[i] = -1.0;
        if (adeg[i]) continue;
        int j;
        double d1, d2;
        kr_nearest(A + (size_t)i * 64, B, nb, bdeg, &j, &d1, &d2);
        if (j < 0) continue;
        if (dist) dist[i] = d1;
        if (second) second[i] = isinf(d2) ? -1.0 : d2;
        if (!(d1 < ratio * d2)) continue;  /* d2 = ∞ passes */
        int back;
        double e1, e2;
        kr_nearest(B + (size_t)j * 64, A, na, adeg, &back, &e1, &e2);
        if (back != i) continue;
        match[i] = j;
        count += 1;
    }
    free(adeg);
    free(bdeg);
    return count;
}

int kazeref_run_batch(const float* imgs, int n, int W, int H, const kazeref_params* p,
                      int64_t cap, int nthreads, int64_t* counts) {
    if (n < 0 || !imgs || !counts) return -1;
    int rc = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
    for (int i = 0; i < n; ++i) {
        kazeref_kp* kps = (kazeref_kp*)malloc(sizeof(kazeref_kp) * (size_t)cap);
        double* desc = (double*)malloc(sizeof(double) * 64 * (size_t)cap);
        counts[i] = kazeref_run(imgs + (size_t)i * W * H, W, H, p, kps, cap, desc, NULL, NULL,
                                NULL, NULL, NULL, NULL);
        if (counts[i] < 0) rc = -1;
        free(kps); free(desc);
    }
    (void)nthreads;
    return rc;
}
