"""CPU checks of the boundary: the C-ABI library builds, loads and exports every symbol include/kaze.h declares,
the ctypes layouts equal the C layouts, the product never routes through the oracle, and argument validation
that happens before any device work.  No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kaze.h")


@pytest.fixture(scope="module")
def K():
    from paper_1706_06750_b200 import build

    build.build()
    import paper_1706_06750_b200 as K

    return K


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kaze_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_binding_names(K):
    assert sorted(K.EXPORTED_SYMBOLS) == _declared()


def test_library_exports_every_declared_symbol(K):
    out = subprocess.run(["nm", "-D", "--defined-only", K.lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kaze_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    lib = K.lib()
    for s in _declared():
        assert hasattr(lib, s)


def test_struct_layouts_match_c(K, tmp_path):
    import ctypes as C

    prog = tmp_path / "sz.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "kaze.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(kaze_params), sizeof(kaze_keypoint),"
        " sizeof(kaze_kernel_stat), offsetof(kaze_params, sigma0), offsetof(kaze_params, max_keypoints),"
        " offsetof(kaze_keypoint, level), offsetof(kaze_keypoint, flags)); printf(\"%zu\\n\", offsetof(kaze_params, tau_max));"
        " return 0;}\n"
    )
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    assert vals == [
        C.sizeof(K.KazeParams), C.sizeof(K.KazeKeypoint), C.sizeof(K.KazeKernelStat),
        K.KazeParams.sigma0.offset, K.KazeParams.max_keypoints.offset,
        K.KazeKeypoint.level.offset, K.KazeKeypoint.flags.offset, K.KazeParams.tau_max.offset,
    ]
    assert vals[1] == 32


def test_defaults_and_status_strings(K):
    p = K.kaze_default_params()
    assert (p.octaves, p.sublevels, p.sigma0, p.k_percentile, p.k_bins) == (4, 4, 1.6, 0.7, 300)
    assert (p.diffusivity, p.threshold, p.edge_ratio, p.ori_windows) == (2, 1e-3, 10.0, 42)
    lib = K.lib()
    for st in (0, -1, -2, -3, -4, -5, -6):
        assert lib.kaze_status_string(st)
    assert K.kaze_abi_version() == 3
    assert (p.scheme, p.tau_max) == (K.SCHEME_AOS, 0.25)


@pytest.mark.parametrize(
    "override,status",
    [
        ({"octaves": 0}, -1), ({"sublevels": 0}, -1), ({"sigma0": 0.0}, -1), ({"sigma0": -1.0}, -1),
        ({"k_percentile": 0.0}, -1), ({"k_percentile": 1.0}, -1), ({"k_bins": 0}, -1), ({"diffusivity": 4}, -1), ({"diffusivity": 0}, -1),
        ({"threshold": -1.0}, -1), ({"max_keypoints": 0}, -1), ({"ori_windows": 65}, -1), ({"max_batch": 0}, -1),
        ({"max_width": 31}, -2), ({"max_height": 16}, -2), ({"scheme": 2}, -1),
        ({"scheme": 1, "tau_max": 0.3}, -1), ({"scheme": 1, "tau_max": 0.0}, -1),
    ],
)
def test_create_rejects_invalid_parameters_before_touching_a_device(K, override, status):
    p = K.kaze_default_params(**override)
    with pytest.raises(K.KazeError) as e:
        K.kaze_create(p, 0)
    assert e.value.status == status


def test_null_arguments_are_rejected(K):
    lib = K.lib()
    assert lib.kaze_create(None, 0, None) == -1
    assert lib.kaze_destroy(None) == 0
    assert lib.kaze_build_scale_space(None, None, 1, 64, 64, 64, None) == -1
    assert lib.kaze_detect(None, None, None, None) == -1
    assert lib.kaze_describe(None, None, None, None, None) == -1
    assert lib.kaze_default_params(None) == -1


def test_product_never_routes_through_the_oracle():
    """The CUDA path and the oracle share no code: no includes, imports or links either way."""
    pkg = os.path.join(ROOT, "paper_1706_06750_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "kazeref" not in txt
                assert not re.search(r"#\s*include\s*[<\"][^>\"]*oracle", txt)
                assert "import oracle" not in txt and "from oracle" not in txt
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_1706_06750_b200" not in txt and "from paper_1706_06750_b200" not in txt
            assert '#include "kaze.h"' not in txt and "include/kaze.h" not in txt and "libkaze_b200" not in txt


def test_fed_cycle_host_schedule_matches_the_oracle(K, oracle_lib):
    """The product's FED cycle (host code inside libkaze_b200.so) against the pinned oracle (P22, A20, A21): the
    same n, the same step sizes (fp32 rounding) and the same κ execution order, for every level transition of the
    KAZE schedule and a few other totals."""
    import numpy as np

    O = oracle_lib
    _, t, _ = O.schedule(4, 4, 1.6)
    totals = list(np.diff(t)) + [0.01, 0.25, 1.0, 3.3, 100.0]
    for T in totals:
        ref = O.fed_cycle(T)
        order = O.fed_order(ref)
        got = K.kaze_fed_cycle(T)
        assert len(got) == len(ref)
        np.testing.assert_allclose(got, ref[order], rtol=2e-7)
        assert abs(float(np.sum(got.astype(np.float64))) / T - 1) < 1e-6
    assert K.lib().kaze_fed_cycle(-1.0, 0.25, None, 0) == -1
    assert K.lib().kaze_fed_cycle(1.0, 0.5, None, 0) == -1
