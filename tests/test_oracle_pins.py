"""Pins for the fp64 CPU oracle (CPU only, no GPU).

The oracle is checked against what the paper and mathematics fix — worked examples printed in
the sources (tests/golden/spec_examples.json, each cited), closed forms, invariants, special
cases that reduce to a textbook or library routine, and brute force on tiny inputs — never
against itself.  Pin ids P1..P21 follow DESIGN.md §5.
"""
import json
import math
import os

import numpy as np
import pytest

import kaze_inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


# ----------------------------------------------------------------------------- P17 schedule
def test_schedule_spec_examples(O):
    for ex in GOLD["schedule"]:
        if "o" in ex:
            sg, t, st = O.schedule(ex["o"] + 1, ex["S"], ex["sigma0"])
            assert sg[ex["o"] * ex["S"] + ex["s"]] == pytest.approx(ex["sigma"], rel=1e-15)
        else:
            sg, t, _ = O.schedule(1, 1, ex["sigma"])
            assert t[0] == pytest.approx(ex["t"], rel=1e-15)


def test_schedule_invariants(O):
    sg, t, st = O.schedule(4, 4, 1.6)
    assert np.all(np.diff(sg) > 0)
    np.testing.assert_allclose(t, sg ** 2 / 2, rtol=0, atol=0)  # Eq. 7 exactly
    # an octave doubles sigma (Eq. 6 read as 2^{o + s/S}); S sublevels per octave
    np.testing.assert_allclose(sg[4:] / sg[:-4], 2.0, rtol=1e-15)
    # s_i = nearest integer to sigma_i, never below 1
    assert np.all(np.abs(st - sg) <= 0.5) and st.min() >= 1


# ----------------------------------------------------------------------------- P1/P2 Gaussian
def test_gaussian_taps_shape(O):
    g = O.gaussian_taps(1.0)
    assert len(g) == 7 and g.sum() == pytest.approx(1.0, abs=1e-15)
    np.testing.assert_array_equal(g, g[::-1])
    assert len(O.gaussian_taps(1.6)) == 11  # r = ceil(3*1.6) = 5
    g01 = O.gaussian_taps(0.1)  # S:L54 delta limit
    assert g01[len(g01) // 2] > 1 - 1e-12


def test_gaussian_blur_impulse_and_corner(O):
    sigma = 1.6
    r = 5
    x = np.arange(-r, r + 1)
    g = np.exp(-x ** 2 / (2 * sigma ** 2))
    g /= g.sum()  # closed form of the sampled normalised Gaussian
    img = np.zeros((31, 29))
    img[15, 11] = 1.0
    out = O.gaussian_blur(img, sigma)
    np.testing.assert_allclose(out[15 - r:15 + r + 1, 11 - r:11 + r + 1], np.outer(g, g), atol=1e-15)
    assert np.abs(out).sum() == pytest.approx(1.0, abs=1e-13)
    # corner impulse with replicate border: out(0,0) = (sum of taps with offset <= 0)^2
    img = np.zeros((20, 20))
    img[0, 0] = 1.0
    out = O.gaussian_blur(img, sigma)
    assert out[0, 0] == pytest.approx(g[: r + 1].sum() ** 2, rel=1e-13)
    # (0, 1): dx in {-r..-1} clamps x+dx to 0 only for dx <= -1
    assert out[0, 1] == pytest.approx(g[: r + 1].sum() * g[:r].sum(), rel=1e-13)


def test_gaussian_blur_invariants(O):
    rng = np.random.default_rng(0)
    c = np.full((16, 16), 0.37)
    np.testing.assert_allclose(O.gaussian_blur(c, 1.6), 0.37, atol=1e-15)
    # linearity and ramp preservation in the interior (symmetric kernel)
    yy, xx = np.mgrid[0:40, 0:40].astype(float)
    ramp = 0.3 * xx - 0.2 * yy + 1.0
    out = O.gaussian_blur(ramp, 1.0)
    np.testing.assert_allclose(out[3:-3, 3:-3], ramp[3:-3, 3:-3], atol=1e-13)
    a, b = rng.random((16, 16)), rng.random((16, 16))
    np.testing.assert_allclose(O.gaussian_blur(2 * a - 3 * b, 1.3),
                               2 * O.gaussian_blur(a, 1.3) - 3 * O.gaussian_blur(b, 1.3), atol=1e-13)


def test_gaussian_semigroup(O):
    """blur(blur(I, a), b) ~ blur(I, sqrt(a^2 + b^2)) on smooth images (1e-3 RMS)."""
    yy, xx = np.mgrid[0:64, 0:64].astype(float)
    img = np.sin(xx / 5.0) * np.cos(yy / 7.0) + 0.5
    two = O.gaussian_blur(O.gaussian_blur(img, 1.0), 1.6)
    one = O.gaussian_blur(img, math.sqrt(1.0 + 1.6 ** 2))
    assert np.sqrt(np.mean((two - one)[10:-10, 10:-10] ** 2)) < 1e-3


# ----------------------------------------------------------------------------- P3 Scharr / Hessian
@pytest.mark.parametrize("s", [1, 2, 3, 5, 8])
def test_scharr_ramp_and_quadratics(O, s):
    yy, xx = np.mgrid[0:64, 0:64].astype(float)
    inner = (slice(2 * s + 1, -2 * s - 1), slice(2 * s + 1, -2 * s - 1))
    np.testing.assert_allclose(O.scharr(xx, s, 0)[inner], 1.0, atol=1e-13)
    np.testing.assert_allclose(O.scharr(xx, s, 1)[inner], 0.0, atol=1e-13)
    np.testing.assert_allclose(O.scharr(yy, s, 1)[inner], 1.0, atol=1e-13)
    np.testing.assert_allclose(O.scharr(np.full((20, 20), 3.0), s, 0), 0.0, atol=0)
    # Hessian closed forms: Ldet = s^4 * det(Hessian) for quadratics
    for ex in GOLD["hessian"]:
        img = (xx ** 2 + yy ** 2) if ex["image"] == "x2+y2" else xx * yy
        img = img / 64.0  # keep values O(1)
        Lx, Ly, Ld = O.hessian(img, s)
        want = ex["factor"] * s ** 4 / 64.0 ** 2 * (1.0 if ex["image"] == "x2+y2" else 1.0)
        np.testing.assert_allclose(Ld[inner], want, rtol=1e-9)
    # first derivatives are s-normalised: Lx = s * d/dx
    Lx, Ly, _ = O.hessian(0.5 * xx + 0.25 * yy, s)
    np.testing.assert_allclose(Lx[inner], 0.5 * s, rtol=1e-12)
    np.testing.assert_allclose(Ly[inner], 0.25 * s, rtol=1e-12)


def test_hessian_mixed_order_is_y_of_x(O):
    """A10: Lxy = Sy[Lx] on the materialised (clamped) Lx — differs from Sx[Ly] only in the 2s band."""
    rng = np.random.default_rng(3)
    img = O.gaussian_blur(rng.random((48, 48)), 2.0)
    s = 3
    lx = O.scharr(img, s, 0)
    ly = O.scharr(img, s, 1)
    dxx, dyy, dxy = O.scharr(lx, s, 0), O.scharr(ly, s, 1), O.scharr(lx, s, 1)
    _, _, Ld = O.hessian(img, s)
    np.testing.assert_allclose(Ld, s ** 4 * (dxx * dyy - dxy ** 2), rtol=1e-12, atol=1e-16)
    dyx = O.scharr(ly, s, 0)
    band = 2 * s
    np.testing.assert_allclose(dxy[band:-band, band:-band], dyx[band:-band, band:-band], atol=1e-14)


# ----------------------------------------------------------------------------- P4 blob scale
def _blob_closed_form(s, v, A):
    """Ldet at the centre of A*exp(-rho^2/2v) for the dilated-Scharr Hessian (derived in DESIGN §5)."""
    e1, e2 = math.exp(-s * s / (2 * v)), math.exp(-2 * s * s / v)
    sm = (118 + 120 * e1 + 18 * e2) / 256.0
    lxx = A * (e2 - 1.0) / (2 * s * s) * sm
    return s ** 4 * lxx * lxx


def test_hessian_blob_closed_form_and_peak_scale(O):
    """BASELINE north_star: 'the Hessian of a synthetic Gaussian blob peaks at its known scale'.
    A blob of std r seen at scale sigma is (r^2/v) exp(-rho^2/2v), v = r^2 + sigma^2 (linear scale
    space); the oracle's Ldet at its centre must equal the closed form, and its argmax over the
    KAZE schedule must be the closed form's argmax (the discrete 'known scale')."""
    sg, _, st = O.schedule(4, 4, 1.6)
    n = 257
    yy, xx = np.mgrid[0:n, 0:n].astype(float) - n // 2
    for r in (4.0, 6.0, 9.0):
        got, want = [], []
        for i in range(16):
            v = r * r + sg[i] ** 2
            A = r * r / v
            img = A * np.exp(-(xx ** 2 + yy ** 2) / (2 * v))
            _, _, Ld = O.hessian(img, int(st[i]))
            got.append(Ld[n // 2, n // 2])
            want.append(_blob_closed_form(int(st[i]), v, A))
        np.testing.assert_allclose(got, want, rtol=1e-10)
        assert int(np.argmax(got)) == int(np.argmax(want))
        # the discrete known scale: levels 3, 6, 9 (closed-form argmax); within 0.6 octave of r —
        # the continuous analogue sigma^4 r^4 / (r^2 + sigma^2)^4 peaks exactly at sigma = r
        assert int(np.argmax(got)) == {4.0: 3, 6.0: 6, 9.0: 9}[r]
        assert abs(math.log2(sg[int(np.argmax(got))] / r)) <= 0.6


# ----------------------------------------------------------------------------- P5 conductivity
def test_conductivity_examples(O):
    yy, xx = np.mgrid[0:40, 0:40].astype(float)
    k = 0.05
    for ex in GOLD["conductivity"]:
        m = ex["grad_over_k"] * k
        img = m * xx  # a ramp stays a ramp of slope m under the symmetric G(1); Scharr gives m
        for g in (1, 2):
            c = O.conductivity(img, k, g)
            np.testing.assert_allclose(c[5:-5, 5:-5], ex[f"g{g}"], rtol=1e-12)
    rng = np.random.default_rng(1)
    L = rng.random((24, 24))
    c1 = O.conductivity(L, 0.04, 2)
    c2 = O.conductivity(3.0 * L, 0.12, 2)  # joint (L, k) scaling invariance
    np.testing.assert_allclose(c1, c2, rtol=1e-12)
    assert c1.min() > 0 and c1.max() <= 1.0


# ----------------------------------------------------------------------------- P6 contrast k
def test_contrast_k_brute_force(O):
    """k from the histogram equals the brute-force order statistic: with the n nonzero interior
    magnitudes sorted, g_(thr) (1-indexed) falls in bin b = min(floor(300 g/hmax), 299), k = hmax(b+1)/300."""
    for seed, (w, h) in [(5, (96, 64)), (6, (64, 64)), (7, (50, 77))]:
        img = kaze_inputs.synth_image(w, h, seed).astype(np.float64)
        L0 = O.gaussian_blur(img, 1.6)
        k, hist, fb = O.contrast_k(L0)
        Ls = O.gaussian_blur(L0, 1.0)
        gx, gy = O.scharr(Ls, 1, 0), O.scharr(Ls, 1, 1)
        g = np.sqrt(gx ** 2 + gy ** 2)[1:-1, 1:-1].ravel()
        hmax = g.max()
        nz = np.sort(g[g > 0])
        thr = int(math.floor(0.7 * len(nz)))
        b = min(int(math.floor(300 * nz[thr - 1] / hmax)), 299)
        assert not fb
        assert k == pytest.approx(hmax * (b + 1) / 300, rel=1e-15)
        assert hist.sum() == len(nz)
        # lambda = 2 scales every magnitude exactly, hence k exactly
        k2, _, _ = O.contrast_k(2.0 * L0)
        assert k2 == 2.0 * k


def test_contrast_k_degenerate(O):
    ex = GOLD["contrast_k"][0]
    k, hist, fb = O.contrast_k(np.full((32, 32), 0.25))
    assert k == ex["constant_image_k"] and fb == ex["fallback"] and hist.sum() == 0


# ----------------------------------------------------------------------------- P10 Thomas / AOS matrix
def test_thomas_vs_dense(O):
    rng = np.random.default_rng(2)
    for n in range(1, 17):
        a, c = -rng.random(n), -rng.random(n)
        b = 1.0 + rng.random(n) + np.abs(a) + np.abs(c)
        d = rng.standard_normal(n)
        M = np.diag(b) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
        np.testing.assert_allclose(O.thomas(a, b, c, d), np.linalg.solve(M, d), rtol=1e-12, atol=1e-14)


def _aos_matrix(cline, tau):
    """I - 2 tau A with A_{j,j+-1} = (c_j + c_{j+-1})/2 and zero row sums (reading A2)."""
    n = len(cline)
    A = np.zeros((n, n))
    for j in range(n - 1):
        w = 0.5 * (cline[j] + cline[j + 1])
        A[j, j + 1] += w
        A[j + 1, j] += w
        A[j, j] -= w
        A[j + 1, j + 1] -= w
    return np.eye(n) - 2 * tau * A


def test_aos_lines_vs_dense(O):
    rng = np.random.default_rng(4)
    for (h, w, tau) in [(5, 7, 0.53), (9, 4, 67.86), (16, 13, 5.99)]:
        L = rng.random((h, w))
        c = rng.uniform(0.05, 1.0, (h, w))
        out, U, V = O.aos_step(L, c, tau)
        for x in range(w):
            np.testing.assert_allclose(U[:, x], np.linalg.solve(_aos_matrix(c[:, x], tau), L[:, x]), rtol=1e-11)
        for y in range(h):
            np.testing.assert_allclose(V[y], np.linalg.solve(_aos_matrix(c[y], tau), L[y]), rtol=1e-11)
        np.testing.assert_allclose(out, 0.5 * (U + V), rtol=0, atol=0)


# ----------------------------------------------------------------------------- P7-P9, P11, P12 AOS
def test_aos_identity_mean_maxprinciple(O):
    rng = np.random.default_rng(5)
    c = rng.uniform(0.01, 1.0, (37, 53))
    out, _, _ = O.aos_step(np.full((37, 53), 0.42), c, 12.0)
    np.testing.assert_allclose(out, 0.42, rtol=1e-14)  # P7
    for tau in (0.53, 5.99, 67.86):
        L = rng.random((37, 53))
        out, U, V = O.aos_step(L, c, tau)
        assert out.mean() == pytest.approx(L.mean(), rel=1e-13)  # P8
        np.testing.assert_allclose(U.sum(axis=0), L.sum(axis=0), rtol=1e-12)
        np.testing.assert_allclose(V.sum(axis=1), L.sum(axis=1), rtol=1e-12)
        assert out.min() >= L.min() - 1e-14 and out.max() <= L.max() + 1e-14  # P9


def test_aos_dct_closed_form(O):
    """P11: with c = 1 every DCT-II mode is an eigenvector of both line operators."""
    H, W = 24, 40
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    c = np.ones((H, W))
    for (k, l, tau) in [(3, 2, 1.5), (7, 0, 20.0), (0, 5, 0.53), (13, 11, 67.86)]:
        mode = np.cos(np.pi * k * (xx + 0.5) / W) * np.cos(np.pi * l * (yy + 0.5) / H)
        lw = 2 - 2 * np.cos(np.pi * k / W)
        lh = 2 - 2 * np.cos(np.pi * l / H)
        out, _, _ = O.aos_step(mode, c, tau)
        np.testing.assert_allclose(out, 0.5 * (1 / (1 + 2 * tau * lw) + 1 / (1 + 2 * tau * lh)) * mode, atol=1e-13)


def test_aos_symmetries(O):
    rng = np.random.default_rng(6)
    L = rng.random((21, 34))
    c = rng.uniform(0.1, 1.0, (21, 34))
    out, _, _ = O.aos_step(L, c, 8.48)
    outT, _, _ = O.aos_step(L.T, c.T, 8.48)
    np.testing.assert_allclose(outT, out.T, rtol=1e-13)
    outR, _, _ = O.aos_step(L[:, ::-1], c[:, ::-1], 8.48)
    np.testing.assert_allclose(outR, out[:, ::-1], rtol=1e-13)


def test_aos_small_steps_approach_gaussian(O):
    """P12 (S:L197 analogue): c = 1, M steps of tau = t/M approach G(sqrt(2t)); error shrinks with M."""
    yy, xx = np.mgrid[0:64, 0:64].astype(float)
    img = np.exp(-((xx - 32) ** 2 + (yy - 32) ** 2) / (2 * 4.0 ** 2))
    t = 4.0
    ref = O.gaussian_blur(img, math.sqrt(2 * t))
    errs = []
    for M in (4, 32):
        L = img.copy()
        for _ in range(M):
            L, _, _ = O.aos_step(L, np.ones_like(L), t / M)
        errs.append(np.sqrt(np.mean((L - ref) ** 2)))
    assert errs[1] < errs[0] and errs[1] < 1e-2


# ----------------------------------------------------------------------------- P19 edge / sub-pixel
def test_refine_spec_examples(O):
    e = GOLD["edge_test"]
    # isotropic peak: D = -(x^2 + y^2) gives Dxx = Dyy = -2, Dxy = 0
    patch = -np.array([[2, 1, 2], [1, 0, 1], [2, 1, 2]], float) + 5.0
    keep, dx, dy = O.refine(patch, e[0]["r"])
    assert keep is e[0]["keep"] and dx == 0.0 and dy == 0.0
    # ridge: Dxx = -10, Dyy = -0.01 -> Tr^2/Det ~ 1002 > 12.1 -> reject
    patch = np.array([[-5.005, -0.005, -5.005], [-5.0, 0.0, -5.0], [-5.005, -0.005, -5.005]]) + 5.0
    keep, _, _ = O.refine(patch, e[1]["r"])
    assert keep is e[1]["keep"]
    assert (-10.01) ** 2 / (10 * 0.01) == pytest.approx(e[1]["ratio_approx"], rel=1e-3)
    # the minimum possible Tr^2/Det is 4 (alpha = beta), i.e. (r+1)^2/r at r = 1
    assert (e[2]["r"] + 1) ** 2 / e[2]["r"] == e[2]["min_ratio"]


@pytest.mark.parametrize("ex", GOLD["subpixel"])
def test_refine_quadratic_recovery(O, ex):
    px, py = ex["peak"]
    yy, xx = np.mgrid[-1:2, -1:2].astype(float)
    patch = 1.0 - (xx - px) ** 2 - (yy - py) ** 2
    keep, dx, dy = O.refine(patch, 10.0)
    assert keep is ex["keep"]
    if keep:
        assert abs(dx - px) < ex["tol"] and abs(dy - py) < ex["tol"]


def test_refine_anisotropic_quadratic(O):
    """Exact recovery for a rotated elliptic quadratic with a cross term (not only the isotropic case)."""
    yy, xx = np.mgrid[-1:2, -1:2].astype(float)
    px, py = -0.35, 0.41
    q = 1.3 * (xx - px) ** 2 + 0.8 * (yy - py) ** 2 + 0.5 * (xx - px) * (yy - py)
    keep, dx, dy = O.refine(2.0 - q, 10.0)
    assert keep and abs(dx - px) < 1e-12 and abs(dy - py) < 1e-12


# ----------------------------------------------------------------------------- P18 extrema
def test_extrema_constant_and_single_blob(O):
    sg, _, st = O.schedule(4, 4, 1.6)
    res = O.run(np.full((64, 64), 0.5, np.float32))
    assert res["count"] == 0 and res["fallback"]
    yy, xx = np.mgrid[0:96, 0:96].astype(float)
    blob = 0.2 + 0.6 * np.exp(-((xx - 47.3) ** 2 + (yy - 48.6) ** 2) / (2 * 2.0 ** 2))
    res = O.run(blob.astype(np.float32), octaves=2, sublevels=2)
    kp = res["kps"]
    assert res["count"] == 1
    assert abs(kp["x"][0] - 47.3) <= 1.0 and abs(kp["y"][0] - 48.6) <= 1.0


def test_extrema_vs_vectorised_scan(O):
    """A second, vectorised statement of the 3x3x3 rule (numpy shifts) gives the same set."""
    sg, _, st = O.schedule(2, 2, 1.6)
    for seed in range(3):
        img = kaze_inputs.synth_image(64, 64, 100 + seed)
        res = O.run(img, octaves=2, sublevels=2, want_levels=True, edge_ratio=0.0)
        D = res["Ldet"]
        N, H, W = D.shape
        found = set()
        for i in range(1, N - 1):
            c = D[i, 1:-1, 1:-1]
            ok = c > 1e-3
            for l in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        if l == dy == dx == 0:
                            continue
                        ok &= c > D[i + l, 1 + dy:H - 1 + dy, 1 + dx:W - 1 + dx]
            for y, x in zip(*np.nonzero(ok)):
                keep, _, _ = O.refine(D[i, y:y + 3, x:x + 3], 0.0)
                if keep:
                    found.add((i, float(D[i, y + 1, x + 1])))
        got = {(int(k["level"]), float(k["response"])) for k in res["kps"]}
        assert res["count"] == len(found) > 0
        assert got == found


# ----------------------------------------------------------------------------- P14 / P15 / P13 invariances
def test_translation_invariance(O):
    base = kaze_inputs.synth_image(48, 48, 77)
    canvas_a = np.full((200, 200), 0.5, np.float32)
    canvas_b = canvas_a.copy()
    canvas_a[76:124, 76:124] = base
    canvas_b[83:131, 69:117] = base
    ra = O.run(canvas_a, octaves=2, sublevels=2)
    rb = O.run(canvas_b, octaves=2, sublevels=2)
    assert ra["k"] == pytest.approx(rb["k"], rel=1e-12)
    assert ra["count"] == rb["count"] > 0
    ka, kb = np.sort(ra["kps"], order=["level", "y", "x"]), np.sort(rb["kps"], order=["level", "y", "x"])
    np.testing.assert_allclose(kb["x"] - ka["x"], -7.0, atol=1e-9)
    np.testing.assert_allclose(kb["y"] - ka["y"], 7.0, atol=1e-9)
    np.testing.assert_allclose(kb["angle"], ka["angle"], atol=1e-9)


def test_offset_invariance(O):
    img = np.round(kaze_inputs.synth_image(80, 64, 9) * 512) / 1024  # values exact in fp32
    ra = O.run(img.astype(np.float32), octaves=2, sublevels=2)
    rb = O.run((img + 0.25).astype(np.float32), octaves=2, sublevels=2)
    assert ra["count"] == rb["count"] > 0
    np.testing.assert_allclose(ra["kps"]["x"], rb["kps"]["x"], atol=1e-9)
    np.testing.assert_allclose(ra["desc"], rb["desc"], atol=1e-9)


def test_rot90_scale_space_equivariance(O):
    img = kaze_inputs.synth_image(72, 56, 11)
    la, ka, _ = O.scale_space(img, octaves=2, sublevels=3)
    lb, kb, _ = O.scale_space(np.ascontiguousarray(np.rot90(img)), octaves=2, sublevels=3)
    assert ka == pytest.approx(kb, rel=1e-12)
    for i in range(la.shape[0]):
        np.testing.assert_allclose(lb[i], np.rot90(la[i]), atol=1e-12)


def _match_by_position(ka, kb, xa, ya):
    """Index into kb of the keypoint at the same level nearest to each mapped position (xa, ya)."""
    return np.array([int(np.argmin(np.hypot(kb["x"] - xa[j], kb["y"] - ya[j]) + 1e6 * (kb["level"] != ka["level"][j])))
                     for j in range(len(ka))])


def test_rot90_orientation_and_descriptor_equivariance(O):
    """P13: under a 90° rotation the first derivatives rotate exactly ((Lx, Ly) ->
    (Ly, -Lx) with clamped borders), the 113-sample disc and the 24x24 grid map onto themselves, and with 48 windows
    (a multiple of 4) the window set is rotation invariant.  So every keypoint maps to x' = y, y' = W-1-x, its angle
    drops by exactly π/2 and its descriptor is unchanged.  (Ldet itself is equivariant only away from the border:
    N_y(N_x L) = N_x(N_y L) holds in the interior but not on the clamped intermediate, so keypoints within 2s_i + 1
    px of the border are excluded.)"""
    img = kaze_inputs.synth_image(150, 110, 31)
    H, W = img.shape
    kw = dict(octaves=3, sublevels=3, ori_windows=48)
    ra, rb = O.run(img, **kw), O.run(np.ascontiguousarray(np.rot90(img)), **kw)
    _, _, st = O.schedule(3, 3, 1.6)
    ka, kb = ra["kps"], rb["kps"]
    s = st[ka["level"]]
    inner = np.minimum(np.minimum(ka["x"], ka["y"]), np.minimum(W - 1 - ka["x"], H - 1 - ka["y"])) >= 2 * s + 1
    assert inner.sum() >= 50 and abs(ra["count"] - rb["count"]) <= (~inner).sum()
    ka, da = ka[inner], ra["desc"][inner]
    xa, ya = ka["y"], W - 1 - ka["x"]
    idx = _match_by_position(ka, kb, xa, ya)
    np.testing.assert_allclose(kb["x"][idx], xa, atol=1e-9)
    np.testing.assert_allclose(kb["y"][idx], ya, atol=1e-9)
    dang = (kb["angle"][idx] - (ka["angle"] - math.pi / 2) + math.pi) % (2 * math.pi) - math.pi
    assert np.max(np.abs(dang)) < 1e-9
    np.testing.assert_allclose(rb["desc"][idx], da, atol=1e-9)


def test_flip_orientation_and_descriptor_signed_permutation(O):
    """P16: a horizontal flip maps (Lx, Ly) -> (-Lx, Ly) exactly (every operator is symmetric and the
    borders clamp), so x' = W-1-x, θ' = π - θ (42 windows: even, so the window set is flip invariant), and the
    sample grid (u, v) of the flipped keypoint lands on (u, -v) of the original with du' = du, dv' = -dv: the
    descriptor is the signed permutation d'[4(4(3-b)+a)+j] = ±d[4(4b+a)+j], minus sign for j = 1 (Σdv)."""
    img = kaze_inputs.synth_image(150, 110, 31)
    W = img.shape[1]
    ra = O.run(img, octaves=3, sublevels=3)
    rc = O.run(np.ascontiguousarray(img[:, ::-1]), octaves=3, sublevels=3)
    assert ra["count"] == rc["count"] > 50
    ka, kc = ra["kps"], rc["kps"]
    idx = _match_by_position(ka, kc, W - 1 - ka["x"], ka["y"])
    assert len(set(idx.tolist())) == len(idx)
    np.testing.assert_allclose(kc["x"][idx], W - 1 - ka["x"], atol=1e-9)
    np.testing.assert_allclose(kc["y"][idx], ka["y"], atol=1e-9)
    dang = (kc["angle"][idx] - (math.pi - ka["angle"]) + math.pi) % (2 * math.pi) - math.pi
    assert np.max(np.abs(dang)) < 1e-9
    perm, sgn = np.zeros(64, int), np.ones(64)
    for b in range(4):
        for a in range(4):
            for j in range(4):
                perm[4 * (4 * b + a) + j] = 4 * (4 * (3 - b) + a) + j
                sgn[4 * (4 * b + a) + j] = -1.0 if j == 1 else 1.0
    np.testing.assert_allclose(rc["desc"][idx][:, perm] * sgn, ra["desc"], atol=1e-9)


# ----------------------------------------------------------------------------- P20 orientation
@pytest.mark.parametrize("theta", [0.0, 0.3, math.pi / 6, 2.0, 4.4, 6.0])
def test_orientation_uniform_gradient(O, theta):
    Lx = np.full((64, 64), math.cos(theta))
    Ly = np.full((64, 64), math.sin(theta))
    ang, deg = O.orientation(Lx, Ly, 31.4, 30.2, 2.3)
    assert not deg
    assert abs(((ang - theta + math.pi) % (2 * math.pi)) - math.pi) < 1e-12


def test_orientation_degenerate_and_windows(O):
    z = np.zeros((32, 32))
    ang, deg = O.orientation(z, z, 16.0, 16.0, 2.0)
    assert ang == 0.0 and deg
    # two populations: a strong direction wins against a weaker one more than pi/3 away
    yy, xx = np.mgrid[0:64, 0:64].astype(float)
    Lx = np.where(xx < 32, 1.0, 0.0) + np.where(xx >= 32, 0.0, 0.0)
    Ly = np.where(xx >= 32, 0.3, 0.0)
    ang, _ = O.orientation(Lx, Ly, 32.0, 32.0, 1.0)
    assert abs(ang) < 1e-12 or abs(ang - 2 * math.pi) < 1e-12


@pytest.mark.parametrize("r1,r2", [((5, 0), (1, 0)), ((3, 4), (0, 2)), ((6, 0), (2, 3)), ((0, -6), (4, 4))])
def test_orientation_gaussian_weight_by_two_impulses(O, r1, r2):
    """P20b (A14): σ = 2 at an integer keypoint puts the 113 samples on pixels 2 px apart, so a field
    that is zero except at two sample pixels is read exactly (bilinear at integer points) by one sample each.  With
    the two gradient directions more than π/3 apart no window holds both, and the longest window sum is the larger
    of w(u, v)·|m|, w = exp(−(u² + v²)/12.5) in σ units (std 2.5σ).  Scaling the second impulse to 0.95 / 1.05 of
    the tie w1·m1 / w2 must flip the winner — this fixes the weight's width and its σ units at these radii."""
    w = lambda u, v: math.exp(-(u * u + v * v) / 12.5)  # noqa: E731
    kx, ky, sigma = 40.0, 41.0, 2.0
    phi1, phi2 = 0.4, 0.4 + 2.2
    for f, want in ((0.95, phi1), (1.05, phi2)):
        Lx, Ly = np.zeros((96, 96)), np.zeros((96, 96))
        m2 = f * w(*r1) / w(*r2)
        for (u, v), m, ph in ((r1, 1.0, phi1), (r2, m2, phi2)):
            Lx[int(ky + sigma * v), int(kx + sigma * u)] = m * math.cos(ph)
            Ly[int(ky + sigma * v), int(kx + sigma * u)] = m * math.sin(ph)
        ang, deg = O.orientation(Lx, Ly, kx, ky, sigma)
        assert not deg and abs(ang - want) < 1e-12, (r1, r2, f, ang, want)


def test_orientation_sample_disc_is_radius_6(O):
    """P20c (A14): the samples are the integer (u, v) with u² + v² <= 36 (113 of them): an impulse at (6, 0) or (0, −6)
    (r² = 36) is seen, one at (1, 6), (4, 5) or (5, 4) (r² = 37, 41, 41) is not — the keypoint is then degenerate."""
    assert sum(1 for u in range(-6, 7) for v in range(-6, 7) if u * u + v * v <= 36) == 113
    for (u, v), seen in (((6, 0), True), ((0, -6), True), ((1, 6), False), ((4, 5), False), ((-5, 4), False)):
        Lx, Ly = np.zeros((96, 96)), np.zeros((96, 96))
        Lx[41 + 2 * v, 40 + 2 * u] = 1.0
        ang, deg = O.orientation(Lx, Ly, 40.0, 41.0, 2.0)
        assert deg == (not seen) and ang == 0.0


# ----------------------------------------------------------------------------- P21 descriptor
def test_descriptor_uniform_field_closed_form(O):
    """Uniform (Lx, Ly) = (1, 0) at angle 0 (and (0, 1) at angle pi/2): du = 1, dv = 0 everywhere,
    so desc[4(4b+a)] = w2(a,b) * S and desc[4(4b+a)+2] = w2(a,b) * S with S = (sum_i exp(-(i-4)^2/12.5))^2."""
    i = np.arange(9)
    S = np.exp(-((i - 4.0) ** 2) / 12.5).sum() ** 2
    want = np.zeros(64)
    for b in range(4):
        for a in range(4):
            w2 = math.exp(-((a - 1.5) ** 2 + (b - 1.5) ** 2) / 4.5)
            want[4 * (4 * b + a)] = w2 * S
            want[4 * (4 * b + a) + 2] = w2 * S
    want /= np.linalg.norm(want)
    one, zero = np.ones((80, 80)), np.zeros((80, 80))
    d = O.descriptor(one, zero, 40.2, 39.7, 1.7, 0.0)
    np.testing.assert_allclose(d, want, atol=1e-14)
    d = O.descriptor(zero, one, 40.2, 39.7, 1.7, math.pi / 2)
    np.testing.assert_allclose(d, want, atol=1e-14)
    assert np.all(O.descriptor(zero, zero, 40.0, 40.0, 2.0, 1.0) == 0)  # degenerate -> zero vector


def test_descriptor_subregion_indexing(O):
    """A field that is nonzero only for v > 0 (rows below the keypoint at angle 0) puts its energy
    in the subregions with b >= 2, and a field nonzero only for u > 0 in a >= 2 (index 4(4b+a)+j)."""
    yy, xx = np.mgrid[0:100, 0:100].astype(float)
    cy = cx = 50.0
    sigma = 1.0
    Lx = np.where(yy > cy + 4, 1.0, 0.0)
    d = O.descriptor(Lx, np.zeros_like(Lx), cx, cy, sigma, 0.0).reshape(4, 4, 4)  # [b, a, j]
    assert np.abs(d[:2]).sum() == 0 and np.abs(d[2:]).sum() > 0
    Lx = np.where(xx > cx + 4, 1.0, 0.0)
    d = O.descriptor(Lx, np.zeros_like(Lx), cx, cy, sigma, 0.0).reshape(4, 4, 4)
    assert np.abs(d[:, :2]).sum() == 0 and np.abs(d[:, 2:]).sum() > 0


def test_descriptor_unit_norm_and_affine_invariance(O):
    img = kaze_inputs.synth_image(96, 80, 21).astype(np.float64)
    ra = O.run(img.astype(np.float32), octaves=2, sublevels=2, want_levels=True)
    assert ra["count"] > 0
    norms = np.linalg.norm(ra["desc"], axis=1)
    np.testing.assert_allclose(norms[norms > 0], 1.0, atol=1e-12)
    # pinned keypoints + angles, derivatives of a*I + b are a times those of I
    k2, d2 = O.describe(3.0 * ra["Lx"], 3.0 * ra["Ly"], ra["kps"], keep_angle=True)
    np.testing.assert_allclose(d2, ra["desc"], atol=1e-12)


def test_bilinear_exact_on_planes(O):
    yy, xx = np.mgrid[0:10, 0:12].astype(float)
    img = 0.7 * xx - 1.3 * yy + 2.0
    for (x, y) in [(3.25, 4.75), (0.0, 0.0), (10.9, 8.1)]:
        assert O.bilinear(img, x, y) == pytest.approx(0.7 * x - 1.3 * y + 2.0, abs=1e-13)
    assert O.bilinear(img, -5.0, 4.0) == pytest.approx(img[4, 0])  # clamped


# ----------------------------------------------------------------------------- P22 FED (Eq. 5, A20)
def test_fed_taus_spec_and_closed_form(O):
    for e in GOLD["fed"]["taus"]:
        np.testing.assert_allclose(O.fed_taus(e["n"], e["tau_max"]), e["taus"], rtol=1e-14)
    for n in range(1, 51):  # Σ τ_j = τ_max n(n+1)/3, all positive
        t = O.fed_taus(n, 0.25)
        assert (t > 0).all()
        assert t.sum() == pytest.approx(0.25 * n * (n + 1) / 3, rel=1e-9)


def test_fed_cycle_spec_and_exact_arrival(O):
    for e in GOLD["fed"]["cycle"]:
        t = O.fed_cycle(e["T"], e["tau_max"])
        assert len(t) == e["n"] and t.sum() == pytest.approx(e["T"], rel=1e-12)
    sg, tt, _ = O.schedule(4, 4, 1.6)
    for T in np.diff(tt):
        t = O.fed_cycle(T, 0.25)
        n = len(t)
        assert 0.25 * n * (n + 1) / 3 >= T * (1 - 1e-12) and 0.25 * (n - 1) * n / 3 < T  # smallest such n
        assert t.sum() == pytest.approx(T, rel=1e-12)


def test_fed_cycle_is_stable_polynomial(O):
    """Eq. 5's point: the whole cycle's amplification prod(1 - τ_j μ) stays in [-1, 1] for every Laplacian
    eigenvalue μ in [0, 2/τ_max] (2-D 4-neighbour, c <= 1) although single steps exceed the explicit limit."""
    for n in (1, 2, 5, 17, 40):
        t = O.fed_taus(n, 0.25)
        assert t.max() > 0.25 or n == 1
        mu = np.linspace(0, 8.0, 20001)
        amp = np.prod(1 - t[:, None] * mu[None, :], axis=0)
        assert np.abs(amp).max() <= 1 + 1e-9


def test_fed_step_dct_closed_form_and_invariants(O):
    """c = 1: every Neumann DCT-II mode is an eigenvector of the 4-neighbour step, eigenvalue
    1 − τ(4 sin²(πk/2W) + 4 sin²(πl/2H)); mass is conserved and the max principle holds for τ ≤ 1/4."""
    H, W = 24, 40
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    c = np.ones((H, W))
    for (k, l, tau) in [(3, 2, 0.2), (7, 0, 0.25), (0, 5, 0.1), (13, 11, 1.7)]:
        mode = np.cos(np.pi * k * (xx + 0.5) / W) * np.cos(np.pi * l * (yy + 0.5) / H)
        lam = 1 - tau * (4 * np.sin(np.pi * k / (2 * W)) ** 2 + 4 * np.sin(np.pi * l / (2 * H)) ** 2)
        np.testing.assert_allclose(O.fed_step(mode, c, tau), lam * mode, atol=1e-13)
    rng = np.random.default_rng(22)
    L = rng.random((H, W))
    cr = rng.uniform(0.0, 1.0, (H, W))
    np.testing.assert_allclose(O.fed_step(np.full((H, W), 0.3), cr, 0.25), 0.3, rtol=1e-15)
    for tau in (0.05, 0.25, 3.0):
        out = O.fed_step(L, cr, tau)
        assert out.sum() == pytest.approx(L.sum(), rel=1e-13)
        if tau <= 0.25:
            assert out.min() >= L.min() - 1e-14 and out.max() <= L.max() + 1e-14


def test_fed_step_vs_dense_graph_laplacian(O):
    """Brute force on a 5x4 grid: the step equals (I + τ A) L with A the weighted graph Laplacian of the
    4-neighbour grid, edge weight ½(c_p + c_q), assembled edge by edge."""
    H, W = 4, 5
    rng = np.random.default_rng(23)
    L, c = rng.random((H, W)), rng.uniform(0.1, 1, (H, W))
    n = H * W
    A = np.zeros((n, n))
    for y in range(H):
        for x in range(W):
            for (yy, xx) in ((y, x + 1), (y + 1, x)):
                if yy < H and xx < W:
                    p, q = y * W + x, yy * W + xx
                    w = 0.5 * (c[y, x] + c[yy, xx])
                    A[p, q] += w
                    A[q, p] += w
                    A[p, p] -= w
                    A[q, q] -= w
    np.testing.assert_allclose(O.fed_step(L, c, 0.21), ((np.eye(n) + 0.21 * A) @ L.ravel()).reshape(H, W), atol=1e-14)


def test_fed_unit_conductivity_is_gaussian(O):
    """c = 1, FED evolution to time t ≈ G(sqrt(2t)), RMS < 1e-2 on a smooth 64×64 image."""
    yy, xx = np.mgrid[0:64, 0:64].astype(float)
    img = np.exp(-((xx - 32) ** 2 + (yy - 32) ** 2) / (2 * 4.0 ** 2))
    t = 4.0
    L = img.copy()
    for tau in O.fed_cycle(t, 0.25):
        L = O.fed_step(L, np.ones_like(L), tau)
    ref = O.gaussian_blur(img, math.sqrt(2 * t))
    assert np.sqrt(np.mean((L - ref) ** 2)) < 1e-2


def test_fed_scale_space_mass_and_agreement_with_aos(O):
    """mass conserved over a full g2 FED pyramid on 128×128; FED and AOS discretise the same PDE, so
    their levels agree to within a fraction of how far each level has evolved."""
    img = kaze_inputs.synth_image(128, 128, 3).astype(np.float64)
    lf, kf, _ = O.scale_space(img, octaves=3, sublevels=4, scheme=1)
    la, ka, _ = O.scale_space(img, octaves=3, sublevels=4, scheme=0)
    assert kf == ka
    m0 = lf[0].sum()
    for i in range(1, lf.shape[0]):
        assert lf[i].sum() == pytest.approx(m0, rel=1e-4)
        # the two schemes differ by their splitting / time errors, far less than the evolution itself
        rms = np.sqrt(np.mean((lf[i] - la[i]) ** 2))
        assert rms < 0.25 * np.sqrt(np.mean((lf[i] - lf[0]) ** 2))
    assert lf.min() >= lf[0].min() - 1e-12 and lf.max() <= lf[0].max() + 1e-12


def test_scale_space_schedule_is_gaussian_at_unit_conductivity(O):
    """P27 (Eqs. 6-7: "filtering for time t = σ²/2 is equivalent to a Gaussian of σ"): with k huge,
    c ≡ 1 and the FED scale space is linear diffusion, so level i must be G(sqrt(σ_i² − σ_0²)) * L_0 — the level has
    evolved for t_i − t_0 in total, i.e. the per-level steps are τ_i = t_i − t_{i−1}.  Each level fits its own
    time clearly better than the neighbouring levels' times (a wrong τ composition, e.g. τ_i = t_i, or an
    off-by-one level misses by far more: checked below for τ_i = t_i)."""
    H = W = 160
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    img = np.full((H, W), 0.3)
    for (cx, cy, s, a) in [(80, 80, 7, 0.5), (62, 95, 4, -0.3), (100, 70, 3, 0.25), (75, 60, 9, 0.2)]:
        img += a * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
    lv, _, _ = O.scale_space(img.astype(np.float32), octaves=3, sublevels=3, k_override=1e6, scheme=1)
    sg, t, _ = O.schedule(3, 3, 1.6)
    rms = lambda a, b: float(np.sqrt(np.mean((a - b) ** 2)))  # noqa: E731
    G = [O.gaussian_blur(lv[0], math.sqrt(sg[i] ** 2 - sg[0] ** 2)) if i else lv[0] for i in range(9)]
    for i in range(1, 9):
        own = rms(lv[i], G[i])
        assert own < 1e-3
        assert own < 0.25 * rms(lv[i], G[i - 1])
        if i + 1 < 9:
            assert own < 0.25 * rms(lv[i], G[i + 1])
        wrong = O.gaussian_blur(lv[0], math.sqrt(2 * t[1:i + 1].sum()))  # τ_i = t_i composition
        assert rms(lv[i], wrong) > 2 * own


def _conv_matrix(H, W, ky, kx):
    """Dense (HW x HW) matrix of the 2-D correlation with taps ky (rows) ⊗ kx (columns), clamped reads (A16)."""
    M = np.zeros((H * W, H * W))
    ry, rx = len(ky) // 2, len(kx) // 2
    for y in range(H):
        for x in range(W):
            for dy in range(-ry, ry + 1):
                for dx in range(-rx, rx + 1):
                    M[y * W + x, min(max(y + dy, 0), H - 1) * W + min(max(x + dx, 0), W - 1)] += ky[dy + ry] * kx[dx + rx]
    return M


def _gauss_taps(sigma):
    r = max(1, math.ceil(3 * sigma))  # A6
    g = np.exp(-np.arange(-r, r + 1) ** 2 / (2 * sigma * sigma))
    return g / g.sum()


def _edge_laplacian(H, W, c, axis):
    """Graph Laplacian of the horizontal (axis 'x') or vertical edges, weight (c_p + c_q)/2 (A2), no border flux."""
    A = np.zeros((H * W, H * W))
    for y in range(H):
        for x in range(W):
            yy, xx = (y, x + 1) if axis == "x" else (y + 1, x)
            if yy < H and xx < W:
                p, q = y * W + x, yy * W + xx
                w = 0.5 * (c[p] + c[q])
                A[p, q] += w
                A[q, p] += w
                A[p, p] -= w
                A[q, q] -= w
    return A


@pytest.mark.parametrize("scheme", [0, 1])
def test_scale_space_composition_vs_dense_brute_force(O, scheme):
    """P28 (A1-A8, A20): brute force on a 12x10 image, whole-image dense
    operators instead of per-line solves and separable passes.  L_0 = G(σ0) L (2-D clamped matrix); for i >= 1
    c_i = g2(|Scharr(G(1) L_{i−1})|) from the PREVIOUS level, τ_i = t_i − t_{i−1} with t = σ²/2, σ_i = σ0·2^{o+s/S};
    AOS: L_i = ½[(I − 2τA_y)⁻¹ + (I − 2τA_x)⁻¹] L_{i−1} by dense solves; FED: L_i = Π_j (I + τ_j (A_x + A_y)) L_{i−1}
    with the cycle's step sizes (pinned by P22).  k is the oracle's histogram value (pinned by P6).  Computing c
    from L_0, or τ_i = t_i, changes the levels by ~1e-2 here; the oracle agrees to ~1e-15."""
    img = kaze_inputs.synth_image(12, 10, 8)
    O_, S_, s0 = 2, 3, 1.6
    lv, k, _ = O.scale_space(img, octaves=O_, sublevels=S_, scheme=scheme)
    H, W = img.shape
    n = H * W
    sg = np.array([s0 * 2.0 ** (o + s / S_) for o in range(O_) for s in range(S_)])
    t = sg ** 2 / 2
    L = [_conv_matrix(H, W, _gauss_taps(s0), _gauss_taps(s0)) @ img.astype(np.float64).ravel()]
    G1 = _conv_matrix(H, W, _gauss_taps(1.0), _gauss_taps(1.0))
    Sx = _conv_matrix(H, W, np.array([3, 10, 3]) / 16, np.array([-1, 0, 1]) / 2)
    Sy = _conv_matrix(H, W, np.array([-1, 0, 1]) / 2, np.array([3, 10, 3]) / 16)
    for i in range(1, O_ * S_):
        Ls = G1 @ L[-1]
        gx, gy = Sx @ Ls, Sy @ Ls
        c = 1.0 / (1.0 + (gx * gx + gy * gy) / (k * k))
        tau = t[i] - t[i - 1]
        Ax, Ay = _edge_laplacian(H, W, c, "x"), _edge_laplacian(H, W, c, "y")
        if scheme == 0:
            L.append(0.5 * (np.linalg.solve(np.eye(n) - 2 * tau * Ay, L[-1]) + np.linalg.solve(np.eye(n) - 2 * tau * Ax, L[-1])))
        else:
            v = L[-1].copy()
            for tj in O.fed_cycle(tau, 0.25):
                v = v + tj * ((Ax + Ay) @ v)
            L.append(v)
    ref = np.array([l.reshape(H, W) for l in L])
    np.testing.assert_allclose(lv, ref, rtol=0, atol=1e-12)
    assert np.max(np.abs(ref[-1] - ref[0])) > 1e-2  # the pyramid really evolves


def test_fed_order_is_permutation_and_stable(O):
    """A21: the order is a κ-permutation; in exact arithmetic the cycle is order independent, so with c ≡ 1 a DCT
    mode must come out scaled by Π_j(1 − τ_j μ) whatever the order — natural order loses ~1e-4 of it in fp64 at
    n = 29 (partial products ~1e12), the chosen order keeps it to rounding."""
    sg, t, _ = O.schedule(4, 4, 1.6)
    for T in np.diff(t):
        taus = O.fed_cycle(T)
        o = O.fed_order(taus)
        assert sorted(o.tolist()) == list(range(len(taus)))
        if len(o) > 1:
            kappa = int(o[1])
            assert math.gcd(kappa, len(o)) == 1 and all(o[m] == (kappa * m) % len(o) for m in range(len(o)))
    # exact spectral result: with c ≡ 1 and Neumann borders the orthonormal DCT-II diagonalises A (scipy.fft)
    from scipy.fft import dctn, idctn
    H, W = 16, 24
    taus = O.fed_cycle(67.86)
    assert len(taus) == 29
    rng = np.random.default_rng(24)
    L0 = rng.random((H, W))
    mu = (4 * np.sin(np.pi * np.arange(H) / (2 * H)) ** 2)[:, None] + (4 * np.sin(np.pi * np.arange(W) / (2 * W)) ** 2)[None, :]
    exact = idctn(dctn(L0, norm="ortho") * np.prod(1 - taus[:, None, None] * mu[None], axis=0), norm="ortho")
    def cycle(order):
        L = L0.copy()
        for j in order:
            L = O.fed_step(L, np.ones_like(L), taus[j])
        return L
    np.testing.assert_allclose(cycle(O.fed_order(taus)), exact, atol=1e-12)
    assert np.abs(cycle(range(29)) - exact).max() > 1e-8  # the natural order is measurably worse


# ----------------------------------------------------------------------------- P23 Weickert diffusivity (A24)
def test_weickert_conductivity_closed_forms(O):
    """g3 = 1 − exp(−3.315/(|∇|/k)^8): on a ramp of slope a the interior gradient is exactly a (G1 and the
    Scharr operator both reproduce linear functions), so c = 1 − e^{−3.315} at k = a and 1 − e^{−3.315/256} at
    k = a/2; a constant image gives c = 1 (the |∇| = 0 limit); g1 / g2 stay e^{−1} / ½ at k = a."""
    a = 0.013
    yy, xx = np.mgrid[0:40, 0:48].astype(float)
    L = a * xx
    inner = (slice(6, -6), slice(6, -6))
    np.testing.assert_allclose(O.conductivity(L, a, 3)[inner], 1 - math.exp(-3.315), rtol=1e-12)
    np.testing.assert_allclose(O.conductivity(L, a / 2, 3)[inner], 1 - math.exp(-3.315 / 256), rtol=1e-12)
    np.testing.assert_allclose(O.conductivity(L, a, 1)[inner], math.exp(-1), rtol=1e-12)
    np.testing.assert_allclose(O.conductivity(L, a, 2)[inner], 0.5, rtol=1e-12)
    np.testing.assert_array_equal(O.conductivity(np.full((20, 30), 0.4), 0.05, 3), 1.0)
    # monotone non-increasing in the slope, bounded in (0, 1]
    cs = [O.conductivity(s * xx, 0.02, 3)[20, 24] for s in (0.001, 0.01, 0.02, 0.03, 0.1)]
    assert all(b <= a_ for a_, b in zip(cs, cs[1:])) and 0 < cs[-1] <= cs[0] <= 1


# ----------------------------------------------------------------------------- P24 exact σ window (A22)
def test_exact_window_radius_and_subset(O):
    assert [O.exact_radius(s) for s in (1, 2, 3, 4, 5, 8, 9, 22)] == [1, 1, 1, 2, 2, 4, 4, 11]
    sg, _, st = O.schedule(4, 4, 1.6)
    img = kaze_inputs.synth_image(160, 120, 1234)
    res = O.run(img, want_levels=True)
    D = res["Ldet"]
    approx, na = O.extrema(D, 4, sg, step=st)
    exact, ne = O.extrema(D, 4, sg, step=st, exact=True)
    assert 0 < ne < na  # "relatively less number of keypoints when using the exact procedure"
    key = lambda k: (int(k["level"]), round(float(k["x"]), 9), round(float(k["y"]), 9))  # noqa: E731
    assert {key(k) for k in exact} <= {key(k) for k in approx}


def test_exact_window_vs_maximum_filter(O):
    """A second statement of the exact rule through a library primitive: scipy's maximum_filter with −inf
    outside the image gives the (2r+1)² window maxima at levels i±1, the 3x3 ring at level i."""
    ndi = pytest.importorskip("scipy.ndimage")
    sg, _, st = O.schedule(3, 3, 1.6)
    for seed in range(2):
        img = kaze_inputs.synth_image(72, 64, 300 + seed)
        res = O.run(img, octaves=3, sublevels=3, want_levels=True, edge_ratio=0.0)
        D = res["Ldet"]
        N, H, W = D.shape
        ring = np.ones((3, 3), bool)
        ring[1, 1] = False
        found = set()
        for i in range(1, N - 1):
            r = O.exact_radius(int(st[i]))
            box = np.ones((2 * r + 1, 2 * r + 1), bool)
            m = np.maximum(ndi.maximum_filter(D[i - 1], footprint=box, mode="constant", cval=-np.inf),
                           ndi.maximum_filter(D[i + 1], footprint=box, mode="constant", cval=-np.inf))
            m = np.maximum(m, ndi.maximum_filter(D[i], footprint=ring, mode="constant", cval=-np.inf))
            ok = (D[i] > 1e-3) & (D[i] > m)
            ok[0, :] = ok[-1, :] = ok[:, 0] = ok[:, -1] = False
            for y, x in zip(*np.nonzero(ok)):
                if O.refine(D[i, y - 1:y + 2, x - 1:x + 2], 0.0)[0]:
                    found.add((i, float(D[i, y, x])))
        got, n = O.extrema(D, 3, sg, step=st, exact=True, edge_ratio=0.0)
        assert n == len(found) > 0
        assert {(int(k["level"]), float(k["response"])) for k in got} == found


def test_exact_window_rejects_a_larger_neighbour_two_pixels_away(O):
    D = np.zeros((3, 24, 24))
    D[1, 10, 10] = 1.0
    D[1, 9:12, 9:12] += 0.5 * np.array([[0.2, 0.5, 0.2], [0.5, 0.0, 0.5], [0.2, 0.5, 0.2]])
    D[2, 10, 12] = 1.5  # outside the 3x3 of level i, inside the 5x5 (r = 2 for step 4)
    sg, st = np.array([1.0, 2.0, 4.0]), np.array([4, 4, 4], np.int32)
    _, na = O.extrema(D, 1, sg, step=st, edge_ratio=0.0)
    _, ne = O.extrema(D, 1, sg, step=st, edge_ratio=0.0, exact=True)
    assert (na, ne) == (1, 0)


# ----------------------------------------------------------------------------- P25 3-D refinement (A23)
def _quad3(x0, y0, s0, A, v0=1.0):
    l, yy, xx = np.mgrid[-1:2, -1:2, -1:2].astype(float)
    d = np.stack([xx - x0, yy - y0, l - s0])
    return v0 - 0.5 * np.einsum("i...,ij,j...->...", d, A, d)


@pytest.mark.parametrize("off", [(0.3, -0.2, 0.25), (-0.45, 0.1, -0.6), (0.0, 0.0, 0.0)])
def test_refine3d_recovers_a_quadratic_peak(O, off):
    """Central differences are exact on quadratics, so the 3-D fit returns the peak of any concave quadratic in
    (x, y, level), cross terms included."""
    A = np.array([[2.0, 0.3, 0.2], [0.3, 1.5, -0.1], [0.2, -0.1, 1.2]])
    keep, dx, dy, ds = O.refine3d(_quad3(*off, A), edge_ratio=0.0)
    assert keep
    np.testing.assert_allclose([dx, dy, ds], off, atol=1e-12)


def test_refine3d_rejections_and_reduction_to_2d(O):
    A = np.diag([2.0, 1.5, 1.2])
    assert not O.refine3d(_quad3(0.2, 0.1, 1.7, A), 0.0)[0]  # |δs| > 1
    assert not O.refine3d(_quad3(1.4, 0.1, 0.0, A), 0.0)[0]  # |δx| > 1
    assert not O.refine3d(np.tile(_quad3(0.2, 0.1, 0.0, A)[1], (3, 1, 1)), 0.0)[0]  # flat in level: singular
    ridge = _quad3(0.1, 0.0, 0.0, np.diag([2.0, 0.002, 1.0]))
    assert not O.refine3d(ridge, 10.0)[0] and O.refine3d(ridge, 0.0)[0]  # the 2-D edge test (A12) still applies
    # no cross terms with the level axis: (δx, δy) equal the 2-D fit of the centre slice
    B = np.array([[2.0, 0.4, 0.0], [0.4, 1.0, 0.0], [0.0, 0.0, 0.9]])
    blk = _quad3(0.35, -0.25, 0.4, B)
    k3, dx, dy, _ = O.refine3d(blk, 10.0)
    k2, ex, ey = O.refine(blk[1], 10.0)
    assert k3 and k2 and abs(dx - ex) < 1e-12 and abs(dy - ey) < 1e-12


def test_refine3d_pipeline_sigma_and_positions(O):
    """With refine3d every keypoint's σ is σ_i·2^{δs/S}, |δs| <= 1, and its position is within 1 px of an
    approximate-procedure extremum of the same level (same candidates, different fit)."""
    sg, _, st = O.schedule(4, 4, 1.6)
    img = kaze_inputs.synth_image(128, 96, 1240)
    r2 = O.run(img)
    r3 = O.run(img, refine3d=1)
    assert r3["count"] > 0
    k = r3["kps"]
    ratio = np.log2(k["sigma"] / sg[k["level"]]) * 4
    assert np.all(np.abs(ratio) <= 1 + 1e-12) and np.any(np.abs(ratio) > 1e-3)
    cand = {(int(a["level"]), int(round(a["response"] * 1e12))) for a in r2["kps"]}
    inter = [(int(a["level"]), int(round(a["response"] * 1e12))) in cand for a in k]
    assert np.mean(inter) > 0.5  # most survive both fits (the candidate sets are identical)


# ----------------------------------------------------------------------------- P26 matcher (A25)
def _units(rng, n, d=64):
    x = rng.normal(size=(n, d))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def test_match_spec_examples(O):
    assert "S:L413" in GOLD["match"]["cite"]
    rng = np.random.default_rng(26)
    A = _units(rng, 15)
    m, d1, _, n = O.match(A, A, 0.8)  # identity, distances 0
    assert n == 15 and np.array_equal(m, np.arange(15)) and np.all(d1 == 0)
    E = np.eye(64)[:2]
    m, _, _, n = O.match(E, E, 1.0)  # orthogonal pair, ratio 1: d1 = 0 < d2 = sqrt(2)
    assert n == 2 and np.array_equal(m, [0, 1])
    A = _units(rng, 20)
    p = rng.permutation(20)
    m, _, _, n = O.match(A, A[p], 0.8)
    assert n == 20 and np.array_equal(p[m], np.arange(20))


def test_match_properties_vs_cdist(O):
    """Distances equal scipy's cdist (a library routine, not the oracle's loop); the mapping is injective;
    shrinking the ratio never adds matches; the first/second distances are the row minima of cdist over the
    non-degenerate columns; degenerate rows never match and are never candidates."""
    sd = pytest.importorskip("scipy.spatial.distance")
    rng = np.random.default_rng(27)
    A = _units(rng, 60)
    B = np.concatenate([A[rng.permutation(60)[:40]] + 0.15 * rng.normal(size=(40, 64)), _units(rng, 30)])
    B /= np.linalg.norm(B, axis=1, keepdims=True)
    B[5] = 0.0  # degenerate
    A[7] = 0.0
    D = sd.cdist(A, B)
    D[:, 5] = np.inf
    prev = None
    for ratio in (1.0, 0.9, 0.8, 0.6, 0.3):
        m, d1, d2, n = O.match(A, B, ratio)
        ok = m >= 0
        assert len(set(m[ok])) == ok.sum() == n  # injective
        assert m[7] == -1 and 5 not in m
        rows = [i for i in range(60) if i != 7]
        srt = np.sort(D[rows], axis=1)
        np.testing.assert_allclose(d1[rows], srt[:, 0], rtol=0, atol=1e-12)
        np.testing.assert_allclose(d2[rows], srt[:, 1], rtol=0, atol=1e-12)
        for i in np.nonzero(ok)[0]:
            j = m[i]
            assert D[i, j] == D[i].min() and d1[i] < ratio * d2[i]
            col = D[:, j].copy()
            col[7] = np.inf
            assert np.argmin(col) == i  # cross-check
        if prev is not None:
            assert set(np.nonzero(ok)[0]) <= prev
        prev = set(np.nonzero(ok)[0])


def test_match_ties_and_edge_cases(O):
    rng = np.random.default_rng(28)
    A = _units(rng, 4)
    B = np.stack([A[1], A[1], A[2], A[3]])  # duplicate nearest: d1 == d2 → the ratio test rejects
    m, d1, d2, _ = O.match(A, B, 1.0)
    assert m[1] == -1 and d1[1] == d2[1] == 0.0
    assert m[2] == 2 and m[3] == 3
    m, d1, d2, n = O.match(A[:1], A[:1], 0.5)  # a single candidate: d2 = ∞ passes any ratio
    assert n == 1 and d2[0] == -1.0
    m, _, _, n = O.match(np.zeros((3, 64)), A, 0.8)
    assert n == 0 and np.all(m == -1)
    m, _, _, n = O.match(A, np.zeros((0, 64)), 0.8)
    assert n == 0 and np.all(m == -1)
