"""B200-native KAZE hot path (arXiv 1706.06750) — thin Python binding over the C ABI of include/kaze.h.

Every step of the path runs in the sm_100a kernels of ``libkaze_b200.so``; this module only marshals
arguments: torch tensors supply device memory and the current CUDA stream, numpy arrays supply host
memory.  There is no CPU fallback: importing works without the library (so the build can be checked on
a CPU-only machine), but every call raises if ``libkaze_b200.so`` is missing or no CUDA device exists.

The functions carry the C names (``kaze_create``, ``kaze_build_scale_space``, ``kaze_detect``,
``kaze_describe``, ...); :class:`Kaze` is a small convenience wrapper over them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "KazeParams", "KazeKeypoint", "KazeKernelStat", "KazeError", "KP_DTYPE", "lib", "lib_path",
    "kaze_default_params", "kaze_create", "kaze_destroy", "kaze_build_scale_space", "kaze_detect",
    "kaze_describe", "kaze_extract", "kaze_extract_host", "kaze_get_k", "kaze_get_level", "kaze_set_level",
    "kaze_set_profiling", "kaze_get_profile", "kaze_reset_profile", "kaze_launch_count", "kaze_abi_version",
    "kaze_fed_cycle", "kaze_match_scratch_bytes", "kaze_match", "kaze_memory_footprint", "KazeMemory", "Kaze", "PLANE_LT", "PLANE_LX", "PLANE_LY", "PLANE_LDET", "PLANE_COND", "FLAG_KEEP_ANGLE", "FLAG_EXACT_WINDOW", "FLAG_REFINE_3D", "FLAG_NO_GRAPHS", "FLAG_ALL_DERIVATIVES", "SCHEME_AOS", "SCHEME_FED",
    "EXPORTED_SYMBOLS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# KAZE_LIB_VARIANT=name loads libkaze_b200.name.so instead (A/B builds from `python -m paper_1706_06750_b200.build
# --variant name -DFLAG...`; experiments only)
_variant = os.environ.get("KAZE_LIB_VARIANT", "")
lib_path = os.path.join(_HERE, f"libkaze_b200.{_variant}.so" if _variant else "libkaze_b200.so")

PLANE_LT, PLANE_LX, PLANE_LY, PLANE_LDET, PLANE_COND = 0, 1, 2, 3, 4
FLAG_KEEP_ANGLE = 1
FLAG_EXACT_WINDOW, FLAG_REFINE_3D = 2, 4
FLAG_NO_GRAPHS = 8  # kaze_extract launches every kernel directly instead of replaying CUDA graphs
FLAG_ALL_DERIVATIVES = 16  # also store (Lx, Ly) of the first and last level (otherwise only their Ldet exists)
SCHEME_AOS, SCHEME_FED = 0, 1

STATUS = {
    0: "ok", -1: "invalid argument", -2: "image too small", -3: "capacity", -4: "state",
    -5: "CUDA error", -6: "out of memory",
}

# Every symbol include/kaze.h declares (checked by tests/test_abi.py against the header and the .so).
EXPORTED_SYMBOLS = [
    "kaze_default_params", "kaze_create", "kaze_destroy", "kaze_build_scale_space", "kaze_detect",
    "kaze_describe", "kaze_extract", "kaze_extract_host", "kaze_get_k", "kaze_get_level", "kaze_set_level",
    "kaze_set_profiling", "kaze_get_profile", "kaze_reset_profile", "kaze_launch_count",
    "kaze_status_string", "kaze_last_error", "kaze_abi_version", "kaze_fed_cycle", "kaze_match_scratch_bytes",
    "kaze_match", "kaze_memory_footprint",
]


class KazeError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str = ""):
        self.status = status
        super().__init__(f"{what}: {STATUS.get(status, status)}" + (f" ({detail})" if detail else ""))


class KazeParams(C.Structure):
    _fields_ = [
        ("max_width", C.c_int32), ("max_height", C.c_int32), ("max_batch", C.c_int32),
        ("octaves", C.c_int32), ("sublevels", C.c_int32),
        ("sigma0", C.c_double), ("k_percentile", C.c_double),
        ("k_bins", C.c_int32), ("diffusivity", C.c_int32),
        ("k_override", C.c_double), ("threshold", C.c_double), ("edge_ratio", C.c_double),
        ("max_keypoints", C.c_int32), ("ori_windows", C.c_int32), ("flags", C.c_int32),
        ("scheme", C.c_int32), ("tau_max", C.c_double),
    ]


class KazeKeypoint(C.Structure):
    _fields_ = [
        ("x", C.c_float), ("y", C.c_float), ("sigma", C.c_float), ("response", C.c_float),
        ("angle", C.c_float), ("level", C.c_int32), ("octave", C.c_int16), ("sublevel", C.c_int16),
        ("flags", C.c_int32),
    ]


KP_DTYPE = np.dtype([
    ("x", "f4"), ("y", "f4"), ("sigma", "f4"), ("response", "f4"), ("angle", "f4"),
    ("level", "i4"), ("octave", "i2"), ("sublevel", "i2"), ("flags", "i4"),
])
assert KP_DTYPE.itemsize == C.sizeof(KazeKeypoint) == 32


class KazeKernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("algo_bytes", C.c_double)]


class KazeMemory(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("evolution", "derivatives", "response", "scratch", "detector", "textures",
                                          "host_path", "pinned_host", "total")]


_lib = None
_vp = C.c_void_p


def lib():
    """Loads libkaze_b200.so (raises loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise RuntimeError(
            f"CUDA extension missing: {lib_path} not built. Run `python -c 'import __graft_entry__ as g; g.build()'`."
        )
    L = C.CDLL(lib_path)
    P = C.POINTER
    L.kaze_default_params.argtypes = [P(KazeParams)]
    L.kaze_create.argtypes = [P(KazeParams), C.c_int, P(_vp)]
    L.kaze_destroy.argtypes = [_vp]
    L.kaze_build_scale_space.argtypes = [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _vp]
    L.kaze_detect.argtypes = [_vp, _vp, _vp, _vp]
    L.kaze_describe.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.kaze_extract.argtypes = [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp, _vp]
    L.kaze_extract_host.argtypes = [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp, _vp]
    L.kaze_get_k.argtypes = [_vp, _vp, _vp]
    L.kaze_get_level.argtypes = [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp]
    L.kaze_set_level.argtypes = [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp]
    L.kaze_set_profiling.argtypes = [_vp, C.c_int32]
    L.kaze_get_profile.argtypes = [_vp, P(KazeKernelStat), C.c_int32, P(C.c_int32)]
    L.kaze_reset_profile.argtypes = [_vp]
    L.kaze_launch_count.argtypes = [_vp]
    L.kaze_memory_footprint.argtypes = [_vp, P(KazeMemory)]
    L.kaze_launch_count.restype = C.c_int64
    L.kaze_status_string.argtypes = [C.c_int]
    L.kaze_status_string.restype = C.c_char_p
    L.kaze_last_error.argtypes = [_vp]
    L.kaze_last_error.restype = C.c_char_p
    L.kaze_abi_version.restype = C.c_int32
    L.kaze_fed_cycle.argtypes = [C.c_double, C.c_double, _vp, C.c_int32]
    L.kaze_fed_cycle.restype = C.c_int32
    L.kaze_match_scratch_bytes.argtypes = [C.c_int32, C.c_int32]
    L.kaze_match_scratch_bytes.restype = C.c_size_t
    L.kaze_match.argtypes = [_vp, C.c_int32, _vp, C.c_int32, C.c_float, _vp, _vp, _vp, C.c_size_t, _vp, _vp]
    for name in EXPORTED_SYMBOLS:
        if name not in ("kaze_launch_count", "kaze_status_string", "kaze_last_error", "kaze_abi_version",
                        "kaze_fed_cycle", "kaze_match_scratch_bytes"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int, what: str, ctx=None):
    if rc != 0:
        detail = lib().kaze_last_error(ctx).decode() if ctx else ""
        raise KazeError(rc, what, detail)


def _ptr(t) -> int:
    """Device or host address of a torch tensor / numpy array (no copies are made here)."""
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None) -> int:
    if stream is not None:
        return int(stream)
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the KAZE path has no CPU fallback")
    return torch.cuda.current_stream().cuda_stream


# ---- C-named functions -----------------------------------------------------------------------------------------
def kaze_default_params(**overrides) -> KazeParams:
    p = KazeParams()
    _check(lib().kaze_default_params(C.byref(p)), "kaze_default_params")
    for k, v in overrides.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


def kaze_create(params: KazeParams, device: int = 0) -> int:
    h = _vp()
    _check(lib().kaze_create(C.byref(params), device, C.byref(h)), "kaze_create")
    return h.value


def kaze_destroy(ctx: int) -> None:
    _check(lib().kaze_destroy(ctx), "kaze_destroy")


def kaze_build_scale_space(ctx: int, imgs, stream=None) -> None:
    """imgs: float32 CUDA tensor [n, h, w] (rows may be padded: the row stride is the pitch)."""
    n, h, w = imgs.shape
    pitch = imgs.stride(1)
    assert imgs.stride(2) == 1 and imgs.stride(0) == pitch * h
    _check(lib().kaze_build_scale_space(ctx, _ptr(imgs), n, w, h, pitch, _stream(stream)), "kaze_build_scale_space", ctx)


def kaze_detect(ctx: int, kps, counts, stream=None) -> None:
    _check(lib().kaze_detect(ctx, _ptr(kps), _ptr(counts), _stream(stream)), "kaze_detect", ctx)


def kaze_describe(ctx: int, kps, counts, desc, stream=None) -> None:
    _check(lib().kaze_describe(ctx, _ptr(kps), _ptr(counts), _ptr(desc), _stream(stream)), "kaze_describe", ctx)


def kaze_extract(ctx: int, imgs, kps, counts, desc, stream=None) -> None:
    n, h, w = imgs.shape
    pitch = imgs.stride(1)
    _check(lib().kaze_extract(ctx, _ptr(imgs), n, w, h, pitch, _ptr(kps), _ptr(counts), _ptr(desc), _stream(stream)),
           "kaze_extract", ctx)


def kaze_extract_host(ctx: int, imgs, kps, counts, desc=None, stream=None) -> None:
    """imgs / kps / counts / desc: host buffers (pinned torch CPU tensors or numpy arrays)."""
    n, h, w = imgs.shape
    pitch = imgs.strides[1] // 4 if isinstance(imgs, np.ndarray) else imgs.stride(1)
    _check(lib().kaze_extract_host(ctx, _ptr(imgs), n, w, h, pitch, _ptr(kps), _ptr(counts),
                                   _ptr(desc) if desc is not None else None, _stream(stream)),
           "kaze_extract_host", ctx)


def kaze_get_k(ctx: int, n: int):
    k = np.zeros(n, np.float32)
    fb = np.zeros(n, np.int32)
    _check(lib().kaze_get_k(ctx, k.ctypes.data, fb.ctypes.data), "kaze_get_k", ctx)
    return k, fb


def kaze_get_level(ctx: int, img: int, level: int, which: int, out, stream=None) -> None:
    _check(lib().kaze_get_level(ctx, img, level, which, _ptr(out), _stream(stream)), "kaze_get_level", ctx)


def kaze_set_level(ctx: int, img: int, level: int, which: int, src, stream=None) -> None:
    _check(lib().kaze_set_level(ctx, img, level, which, _ptr(src), _stream(stream)), "kaze_set_level", ctx)


def kaze_set_profiling(ctx: int, enable: bool) -> None:
    _check(lib().kaze_set_profiling(ctx, int(enable)), "kaze_set_profiling", ctx)


def kaze_reset_profile(ctx: int) -> None:
    _check(lib().kaze_reset_profile(ctx), "kaze_reset_profile", ctx)


def kaze_get_profile(ctx: int) -> dict:
    arr = (KazeKernelStat * 32)()
    n = C.c_int32()
    _check(lib().kaze_get_profile(ctx, arr, 32, C.byref(n)), "kaze_get_profile", ctx)
    return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].total_ms, "bytes": arr[i].algo_bytes}
            for i in range(n.value)}


def kaze_launch_count(ctx: int) -> int:
    return int(lib().kaze_launch_count(ctx))


def kaze_memory_footprint(ctx: int) -> dict:
    """Device bytes the context holds, by role (include/kaze.h kaze_memory)."""
    m = KazeMemory()
    _check(lib().kaze_memory_footprint(ctx, C.byref(m)), "kaze_memory_footprint", ctx)
    return {n: int(getattr(m, n)) for n, _ in KazeMemory._fields_}


def kaze_abi_version() -> int:
    return int(lib().kaze_abi_version())


def kaze_match_scratch_bytes(na: int, nb: int) -> int:
    return int(lib().kaze_match_scratch_bytes(na, nb))


def kaze_match(desc_a, desc_b, ratio: float = 0.8, scratch=None, stream=None):
    """desc_a [na, 64], desc_b [nb, 64]: float32 CUDA tensors → (match [na] int32, dist [na] float32,
    stats [2] int32 = [matches, rows rescanned exactly]).  All on the device; nothing is synchronised."""
    import torch

    na, nb = int(desc_a.shape[0]), int(desc_b.shape[0])
    a = desc_a.contiguous()
    b = desc_b.contiguous()
    dev = a.device
    match = torch.empty(na, dtype=torch.int32, device=dev)
    dist = torch.empty(na, dtype=torch.float32, device=dev)
    stats = torch.zeros(2, dtype=torch.int32, device=dev)
    need = kaze_match_scratch_bytes(na, nb)
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    _check(lib().kaze_match(_ptr(a) if na else None, na, _ptr(b) if nb else None, nb, ratio, _ptr(match),
                            _ptr(dist), _ptr(scratch), scratch.numel(), _ptr(stats), _stream(stream)), "kaze_match")
    return match, dist, stats


def kaze_fed_cycle(T: float, tau_max: float = 0.25) -> np.ndarray:
    """Host-only: the FED cycle's step sizes in execution order for a level transition of total time T."""
    n = int(lib().kaze_fed_cycle(T, tau_max, None, 0))
    if n <= 0:
        raise KazeError(n, "kaze_fed_cycle")
    out = np.zeros(n, np.float32)
    lib().kaze_fed_cycle(T, tau_max, out.ctypes.data, n)
    return out


# ---- convenience wrapper ---------------------------------------------------------------------------------------
class Kaze:
    """One context on one device.  Outputs are torch tensors on that device."""

    def __init__(self, width: int, height: int, batch: int = 1, device: int = 0, **params):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the KAZE path has no CPU fallback")
        self.params = kaze_default_params(max_width=width, max_height=height, max_batch=batch, **params)
        self.device = device
        self.ctx = kaze_create(self.params, device)
        self.N = self.params.octaves * self.params.sublevels
        self.cap = self.params.max_keypoints

    def close(self):
        if getattr(self, "ctx", None):
            kaze_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc_outputs(self, n: int):
        import torch

        dev = torch.device("cuda", self.device)
        kps = torch.zeros((n, self.cap, 8), dtype=torch.int32, device=dev)  # 32-byte records
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        desc = torch.zeros((n, self.cap, 64), dtype=torch.float32, device=dev)
        return kps, counts, desc

    def extract(self, imgs):
        """imgs: [n, h, w] float32 CUDA tensor → (kps [n, cap, 8] int32 records, counts [n], desc [n, cap, 64])."""
        kps, counts, desc = self.alloc_outputs(imgs.shape[0])
        kaze_extract(self.ctx, imgs, kps, counts, desc)
        return kps, counts, desc

    @staticmethod
    def keypoints_numpy(kps, counts, cap: int | None = None) -> list[np.ndarray]:
        """Device records → one structured numpy array (KP_DTYPE) per image, truncated to the counts."""
        k = kps.detach().cpu().numpy() if not isinstance(kps, np.ndarray) else kps
        c = counts.detach().cpu().numpy() if not isinstance(counts, np.ndarray) else counts
        k = np.ascontiguousarray(k).view(KP_DTYPE).reshape(k.shape[0], -1)
        cap = k.shape[1] if cap is None else cap
        return [k[i, : min(int(c[i]), cap)] for i in range(k.shape[0])]
