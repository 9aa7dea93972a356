"""ctypes wrapper around the fp64 C oracle (``oracle/kazeref.c``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_1706_06750_b200``) never imports it and shares no code with it.

Every function returns numpy float64 arrays; images are (H, W) row-major.  Citations of the
paper passages each function follows are in ``kazeref.h`` / ``kazeref.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libkazeref.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -O2, no fast-math, OpenMP over images only)."""
    src = os.path.join(_HERE, "kazeref.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "kazeref.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-o", _SO, src, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


class Params(C.Structure):
    _fields_ = [
        ("octaves", C.c_int32),
        ("sublevels", C.c_int32),
        ("sigma0", C.c_double),
        ("k_percentile", C.c_double),
        ("k_bins", C.c_int32),
        ("diffusivity", C.c_int32),
        ("k_override", C.c_double),
        ("threshold", C.c_double),
        ("edge_ratio", C.c_double),
        ("ori_windows", C.c_int32),
        ("keep_angle", C.c_int32),
        ("scheme", C.c_int32),
        ("tau_max", C.c_double),
        ("exact_window", C.c_int32),
        ("refine3d", C.c_int32),
    ]


class KP(C.Structure):
    _fields_ = [
        ("x", C.c_double),
        ("y", C.c_double),
        ("sigma", C.c_double),
        ("response", C.c_double),
        ("angle", C.c_double),
        ("level", C.c_int32),
        ("octave", C.c_int32),
        ("sublevel", C.c_int32),
        ("degenerate", C.c_int32),
    ]


KP_DTYPE = np.dtype(
    [
        ("x", "f8"), ("y", "f8"), ("sigma", "f8"), ("response", "f8"), ("angle", "f8"),
        ("level", "i4"), ("octave", "i4"), ("sublevel", "i4"), ("degenerate", "i4"),
    ]
)
assert KP_DTYPE.itemsize == C.sizeof(KP)

_lib = None
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.kazeref_default_params.argtypes = [C.POINTER(Params)]
        L.kazeref_schedule.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp, C.POINTER(C.c_int32)]
        L.kazeref_gaussian_taps.argtypes = [C.c_double, _dp, C.POINTER(C.c_int32)]
        L.kazeref_gaussian_blur.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
        L.kazeref_scharr.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.kazeref_contrast_k.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_int, _dp,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.kazeref_conductivity.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_int, _dp]
        L.kazeref_thomas.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.kazeref_aos_step.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp]
        L.kazeref_scale_space.argtypes = [_fp, C.c_int, C.c_int, C.POINTER(Params), _dp, _dp,
                                          C.POINTER(C.c_int32)]
        L.kazeref_hessian.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.kazeref_refine.argtypes = [_dp, C.c_double, _dp, _dp]
        L.kazeref_extrema.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_double,
                                      C.c_double, C.POINTER(KP), C.c_int64]
        L.kazeref_extrema.restype = C.c_int64
        L.kazeref_extrema2.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.POINTER(C.c_int32),
                                       C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(KP), C.c_int64]
        L.kazeref_extrema2.restype = C.c_int64
        L.kazeref_refine3d.argtypes = [_dp, C.c_double, _dp, _dp, _dp]
        L.kazeref_match.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_double, C.POINTER(C.c_int32), _dp, _dp]
        L.kazeref_match.restype = C.c_int64
        L.kazeref_exact_radius.argtypes = [C.c_int]
        L.kazeref_bilinear.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double]
        L.kazeref_bilinear.restype = C.c_double
        L.kazeref_orientation.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_int, C.POINTER(C.c_int32)]
        L.kazeref_orientation.restype = C.c_double
        L.kazeref_descriptor.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_double, _dp]
        L.kazeref_describe.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.POINTER(KP),
                                       C.c_int64, C.c_int, C.c_int, _dp]
        L.kazeref_run.argtypes = [_fp, C.c_int, C.c_int, C.POINTER(Params), C.POINTER(KP),
                                  C.c_int64, _dp, _dp, C.POINTER(C.c_int32), _dp, _dp, _dp, _dp]
        L.kazeref_run.restype = C.c_int64
        L.kazeref_fed_taus.argtypes = [C.c_int, C.c_double, _dp]
        L.kazeref_fed_cycle.argtypes = [C.c_double, C.c_double, _dp, C.c_int]
        L.kazeref_fed_order.argtypes = [_dp, C.c_int, C.POINTER(C.c_int32)]
        L.kazeref_fed_step.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, _dp]
        L.kazeref_run_batch.argtypes = [_fp, C.c_int, C.c_int, C.c_int, C.POINTER(Params),
                                        C.c_int64, C.c_int, C.POINTER(C.c_int64)]
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _chk(rc):
    if rc < 0:
        raise ValueError(f"oracle call failed (rc={rc})")
    return rc


def params(**kw) -> Params:
    p = Params()
    lib().kazeref_default_params(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


def schedule(O: int = 4, S: int = 4, sigma0: float = 1.6):
    N = O * S
    sg, t = np.zeros(N), np.zeros(N)
    st = np.zeros(N, np.int32)
    _chk(lib().kazeref_schedule(O, S, sigma0, _d(sg), _d(t), st.ctypes.data_as(C.POINTER(C.c_int32))))
    return sg, t, st


def gaussian_taps(sigma: float) -> np.ndarray:
    r = C.c_int32()
    _chk(lib().kazeref_gaussian_taps(sigma, None, C.byref(r)))
    taps = np.zeros(2 * r.value + 1)
    lib().kazeref_gaussian_taps(sigma, _d(taps), C.byref(r))
    return taps


def gaussian_blur(img, sigma: float) -> np.ndarray:
    a = _f64(img)
    out = np.empty_like(a)
    _chk(lib().kazeref_gaussian_blur(_d(a), a.shape[1], a.shape[0], sigma, _d(out)))
    return out


def scharr(img, s: int, direction: int) -> np.ndarray:
    a = _f64(img)
    out = np.empty_like(a)
    _chk(lib().kazeref_scharr(_d(a), a.shape[1], a.shape[0], s, direction, _d(out)))
    return out


def contrast_k(L0, perc: float = 0.7, bins: int = 300):
    a = _f64(L0)
    k = C.c_double()
    hist = np.zeros(bins, np.int64)
    fb = C.c_int32()
    _chk(lib().kazeref_contrast_k(_d(a), a.shape[1], a.shape[0], perc, bins, C.byref(k),
                                  hist.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(fb)))
    return k.value, hist, bool(fb.value)


def conductivity(L, k: float, diffusivity: int = 2) -> np.ndarray:
    a = _f64(L)
    out = np.empty_like(a)
    _chk(lib().kazeref_conductivity(_d(a), a.shape[1], a.shape[0], k, diffusivity, _d(out)))
    return out


def thomas(a, b, c, d) -> np.ndarray:
    a, b, c, d = (_f64(v) for v in (a, b, c, d))
    x = np.empty_like(d)
    _chk(lib().kazeref_thomas(len(d), _d(a), _d(b), _d(c), _d(d), _d(x)))
    return x


def aos_step(L, c, tau: float):
    """Returns (L_new, U, V)."""
    L, c = _f64(L), _f64(c)
    out, U, V = np.empty_like(L), np.empty_like(L), np.empty_like(L)
    _chk(lib().kazeref_aos_step(_d(L), _d(c), L.shape[1], L.shape[0], tau, _d(out), _d(U), _d(V)))
    return out, U, V


def scale_space(img, **kw):
    """Returns (levels[N,H,W], k, fallback)."""
    im = np.ascontiguousarray(img, dtype=np.float32)
    p = params(**kw)
    H, W = im.shape
    N = p.octaves * p.sublevels
    lv = np.empty((N, H, W))
    k = C.c_double()
    fb = C.c_int32()
    _chk(lib().kazeref_scale_space(im.ctypes.data_as(_fp), W, H, C.byref(p), _d(lv), C.byref(k), C.byref(fb)))
    return lv, k.value, bool(fb.value)


def fed_taus(n: int, tau_max: float = 0.25) -> np.ndarray:
    t = np.zeros(n)
    _chk(lib().kazeref_fed_taus(n, tau_max, _d(t)))
    return t


def fed_cycle(T: float, tau_max: float = 0.25) -> np.ndarray:
    n = _chk(lib().kazeref_fed_cycle(T, tau_max, None, 0))
    t = np.zeros(n)
    lib().kazeref_fed_cycle(T, tau_max, _d(t), n)
    return t


def fed_order(taus) -> np.ndarray:
    t = _f64(taus)
    o = np.zeros(len(t), np.int32)
    _chk(lib().kazeref_fed_order(_d(t), len(t), o.ctypes.data_as(C.POINTER(C.c_int32))))
    return o


def fed_step(L, c, tau: float) -> np.ndarray:
    a, b = _f64(L), _f64(c)
    out = np.empty_like(a)
    _chk(lib().kazeref_fed_step(_d(a), _d(b), a.shape[1], a.shape[0], tau, _d(out)))
    return out


def hessian(L, s: int):
    """Returns (Lx, Ly, Ldet)."""
    a = _f64(L)
    Lx, Ly, Ld = np.empty_like(a), np.empty_like(a), np.empty_like(a)
    _chk(lib().kazeref_hessian(_d(a), a.shape[1], a.shape[0], s, _d(Lx), _d(Ly), _d(Ld)))
    return Lx, Ly, Ld


def refine(patch, edge_ratio: float = 10.0):
    """Returns (keep, dx, dy) for a 3x3 response patch (row = y)."""
    p = _f64(np.asarray(patch).reshape(9))
    dx, dy = C.c_double(np.nan), C.c_double(np.nan)
    keep = lib().kazeref_refine(_d(p), edge_ratio, C.byref(dx), C.byref(dy))
    return bool(keep), dx.value, dy.value


def refine3d(block, edge_ratio: float = 10.0):
    """Returns (keep, dx, dy, ds) for a 3x3x3 response block [level][row][col]."""
    p = _f64(np.asarray(block).reshape(27))
    dx, dy, ds = C.c_double(np.nan), C.c_double(np.nan), C.c_double(np.nan)
    keep = lib().kazeref_refine3d(_d(p), edge_ratio, C.byref(dx), C.byref(dy), C.byref(ds))
    return bool(keep), dx.value, dy.value, ds.value


def exact_radius(step: int) -> int:
    return int(lib().kazeref_exact_radius(step))


def extrema(Ldet, S: int, sigma, threshold: float = 1e-3, edge_ratio: float = 10.0, cap: int = 1 << 20,
            step=None, exact: bool = False, refine3d: bool = False):
    Ld = _f64(Ldet)
    N, H, W = Ld.shape
    sg = _f64(sigma)
    st = np.ascontiguousarray(step if step is not None else np.ones(N), dtype=np.int32)
    buf = np.zeros(cap, KP_DTYPE)
    n = lib().kazeref_extrema2(_d(Ld), N, W, H, S, _d(sg), st.ctypes.data_as(C.POINTER(C.c_int32)), threshold,
                               edge_ratio, int(exact), int(refine3d), buf.ctypes.data_as(C.POINTER(KP)), cap)
    _chk(n)
    return buf[: min(n, cap)].copy(), n


def match(A, B, ratio: float = 0.8):
    """Brute-force matcher (A25) → (match[na] (b or -1), d1[na], d2[na], count)."""
    a = _f64(np.asarray(A).reshape(-1, 64))
    b = _f64(np.asarray(B).reshape(-1, 64))
    na, nb = len(a), len(b)
    m = np.zeros(na, np.int32)
    d1, d2 = np.zeros(na), np.zeros(na)
    n = lib().kazeref_match(_d(a), na, _d(b), nb, ratio, m.ctypes.data_as(C.POINTER(C.c_int32)), _d(d1), _d(d2))
    _chk(n)
    return m, d1, d2, int(n)


def bilinear(img, x: float, y: float) -> float:
    a = _f64(img)
    return lib().kazeref_bilinear(_d(a), a.shape[1], a.shape[0], x, y)


def orientation(Lx, Ly, x, y, sigma, nwin: int = 42):
    a, b = _f64(Lx), _f64(Ly)
    deg = C.c_int32()
    ang = lib().kazeref_orientation(_d(a), _d(b), a.shape[1], a.shape[0], x, y, sigma, nwin, C.byref(deg))
    return ang, bool(deg.value)


def descriptor(Lx, Ly, x, y, sigma, angle) -> np.ndarray:
    a, b = _f64(Lx), _f64(Ly)
    d = np.zeros(64)
    lib().kazeref_descriptor(_d(a), _d(b), a.shape[1], a.shape[0], x, y, sigma, angle, _d(d))
    return d


def describe(Lx, Ly, kps: np.ndarray, nwin: int = 42, keep_angle: bool = False):
    """Lx, Ly: [N,H,W]; kps: KP_DTYPE array (modified copy returned) → (kps, desc[n,64])."""
    a, b = _f64(Lx), _f64(Ly)
    N, H, W = a.shape
    k = np.ascontiguousarray(kps.copy(), dtype=KP_DTYPE)
    desc = np.zeros((len(k), 64))
    _chk(lib().kazeref_describe(_d(a), _d(b), N, W, H, k.ctypes.data_as(C.POINTER(KP)), len(k), nwin,
                                int(keep_angle), _d(desc)))
    return k, desc


def run(img, cap: int = 1 << 18, want_levels: bool = False, **kw):
    """Full oracle path on one float32 image (H, W).

    Returns dict(kps, desc, count, k, fallback[, levels, Lx, Ly, Ldet])."""
    im = np.ascontiguousarray(img, dtype=np.float32)
    p = params(**kw)
    H, W = im.shape
    N = p.octaves * p.sublevels
    kps = np.zeros(cap, KP_DTYPE)
    desc = np.zeros((cap, 64))
    k = C.c_double()
    fb = C.c_int32()
    out = {}
    if want_levels:
        for name in ("levels", "Lx", "Ly", "Ldet"):
            out[name] = np.empty((N, H, W))
    ptr = lambda n: _d(out[n]) if want_levels else None  # noqa: E731
    n = lib().kazeref_run(im.ctypes.data_as(_fp), W, H, C.byref(p), kps.ctypes.data_as(C.POINTER(KP)),
                          cap, _d(desc), C.byref(k), C.byref(fb), ptr("levels"), ptr("Lx"), ptr("Ly"),
                          ptr("Ldet"))
    _chk(n)
    m = min(n, cap)
    out.update(kps=kps[:m].copy(), desc=desc[:m].copy(), count=int(n), k=k.value, fallback=bool(fb.value))
    return out


def run_batch(imgs, cap: int = 1 << 17, nthreads: int = 1, **kw) -> np.ndarray:
    """Full path on a batch [n, H, W] with OpenMP over images; returns keypoint counts."""
    im = np.ascontiguousarray(imgs, dtype=np.float32)
    n, H, W = im.shape
    p = params(**kw)
    counts = np.zeros(n, np.int64)
    _chk(lib().kazeref_run_batch(im.ctypes.data_as(_fp), n, W, H, C.byref(p), cap, nthreads,
                                 counts.ctypes.data_as(C.POINTER(C.c_int64))))
    return counts
