"""GPU-vs-oracle parity at the instantiations the headline bench runs, and the paths round 1 left untested (needs a
B200).  Every call goes through the C ABI (ctypes -> libkaze_b200.so).

* 1920x1200 scale space in the bench launch configuration (32 images per launch, kaze_extract replaying the chunk
  as a CUDA graph, k estimated on the device), AOS and FED: every level of the first and last image within 1e-4
  relative of the oracle's fp64 levels, run with the GPU's k (itself in the oracle's histogram bin);
  this is the only configuration that instantiates the TMA-staged column pass k_aos_cols_tma<8,19,512,2>
  (832 < H <= 1216 with the 1088 < H rung) and k_aos_rows_cta<15,4> (1792 < W <= 1920).
* Hessian stage-isolated at 1920x1200, O = S = 4 (steps 2, 3, 4, 5, 6, 8, 9, 11, 13, 15, 18, 22: both column-block
  widths of the fused kernel), and at O = 5 (steps up to 43: the two-pass form for s > 32).
* The generic prefilter (σ0 = 1.2 and 2.5; σ0 = 1.6 takes the radius-5 kernel) and the g1 diffusivity (Eq. 3).
* CUDA-graph replay across image sizes A, A, B, B, B, A (one texture table per size).
* Descriptor of keypoints at levels without materialised derivatives.
* rot90 equivariance of the GPU path itself (P13 on the device).
Tolerances as tests/test_gpu_parity.py (BASELINE north_star).
"""
import math

import numpy as np
import pytest

import kaze_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1706_06750_b200 as K  # noqa: E402
from test_gpu_parity import gpu_levels, make, match_keypoints, oracle_run, rel_err  # noqa: E402


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


# ------------------------------------------------------------------------------------------- headline scale space
@pytest.mark.slow
@pytest.mark.parametrize("scheme", [0, 1])
def test_levels_1920x1200_in_bench_launch_configuration(O, scheme):
    imgs = kaze_inputs.synth_batch(32, 1920, 1200, distinct=2)
    kz = make(1920, 1200, batch=32, max_keypoints=32768, scheme=scheme)
    dimg = torch.from_numpy(imgs).cuda()
    out = kz.alloc_outputs(32)
    for _ in range(3):  # direct, captured, replayed: the levels read below come from the graph replay
        K.kaze_extract(kz.ctx, dimg, *out)
    torch.cuda.synchronize()
    kg, fb = K.kaze_get_k(kz.ctx, 32)
    for i in (0, 31):
        # k: the device histogram picks the oracle's bin (k = hmax (b+1)/300, hmax differs by fp32 rounding)
        L0 = O.gaussian_blur(imgs[i].astype(np.float64), 1.6)
        kref, _, _ = O.contrast_k(L0)
        assert abs(kg[i] / kref - 1) < 1e-5 and fb[i] == 0, (i, kg[i], kref)
        ref, _, _ = O.scale_space(imgs[i], k_override=float(kg[i]), scheme=scheme)
        lv = gpu_levels(kz, 16, img=i)
        assert rel_err(lv[0], ref[0]) < 2e-6
        for lvl in range(16):
            e = rel_err(lv[lvl], ref[lvl])
            assert e <= 1e-4, (scheme, i, lvl, e)
        for lvl in range(1, 16):  # mean preserved per step on the GPU too
            assert abs(lv[lvl].mean() / lv[lvl - 1].mean() - 1) < 1e-5
    kz.close()


# ------------------------------------------------------------------------------------------- Hessian at every step
def _hessian_stage_isolated(O, kz, imgs_idx, levels, st, n_levels):
    kps = torch.zeros((kz.batch, kz.cap, 8), dtype=torch.int32, device="cuda")
    counts = torch.zeros(kz.batch, dtype=torch.int32, device="cuda")
    for i, lv in zip(imgs_idx, levels):
        for lvl in range(n_levels):
            K.kaze_set_level(kz.ctx, i, lvl, K.PLANE_LT, torch.from_numpy(lv[lvl].astype(np.float32)).cuda())
    K.kaze_detect(kz.ctx, kps, counts)
    torch.cuda.synchronize()
    worst = 0.0
    for i, lv in zip(imgs_idx, levels):
        Lx, Ly = gpu_levels(kz, n_levels, K.PLANE_LX, img=i), gpu_levels(kz, n_levels, K.PLANE_LY, img=i)
        Ld = gpu_levels(kz, n_levels, K.PLANE_LDET, img=i)
        for lvl in range(n_levels):
            rx, ry, rd = O.hessian(lv[lvl].astype(np.float32).astype(np.float64), int(st[lvl]))
            ex, ey, ed = rel_err(Lx[lvl], rx), rel_err(Ly[lvl], ry), rel_err(Ld[lvl], rd)
            assert ex < 1e-5 and ey < 1e-5, (i, lvl, int(st[lvl]), ex, ey)
            assert ed < 1e-4, (i, lvl, int(st[lvl]), ed)
            worst = max(worst, ed)
    return kps, counts, worst


@pytest.mark.slow
def test_hessian_stage_isolated_1920x1200_all_steps(O):
    """The fused Hessian in the bench configuration (batch of 32, every level of two images injected from the
    oracle): steps 2..22 cover both column-block widths (224 for s <= 16, 192 above) and every template case the
    headline instantiates; Lx, Ly < 1e-5 and Ldet < 1e-4 relative per level; the keypoints of image 0 equal the
    oracle's extrema of the GPU's own Ldet."""
    imgs = kaze_inputs.synth_batch(32, 1920, 1200, distinct=2)
    sg, _, st = O.schedule(4, 4, 1.6)
    assert sorted(set(st.tolist())) == [2, 3, 4, 5, 6, 8, 9, 11, 13, 15, 18, 22]
    kz = make(1920, 1200, batch=32, max_keypoints=32768, flags=K.FLAG_ALL_DERIVATIVES)
    kz.batch = 32
    dimg = torch.from_numpy(imgs).cuda()
    out = kz.alloc_outputs(32)
    K.kaze_extract(kz.ctx, dimg, *out)  # builds all 32 images (the chunk geometry the bench uses)
    levels = [O.scale_space(imgs[i], k_override=0.033)[0] for i in (0, 31)]
    kps, counts, _ = _hessian_stage_isolated(O, kz, (0, 31), levels, st, 16)
    Ld = gpu_levels(kz, 16, K.PLANE_LDET, img=0)
    kref, nref = O.extrema(Ld, 4, sg)
    got = K.Kaze.keypoints_numpy(kps, counts)[0]
    frac, _ = match_keypoints(kref, got, tol=1e-3)
    assert abs(int(counts[0]) - nref) <= max(2, 0.002 * nref) and frac >= 0.995, (int(counts[0]), nref, frac)
    kz.close()


def test_hessian_two_pass_for_steps_above_32(O):
    """O = 5, S = 4: σ_19 = 1.6·2^4.75 ≈ 43 → s = 43 > 32, so detect runs the two chain passes (hess_first +
    hess_det) for every level; Lx, Ly, Ldet vs the oracle on injected levels, and keypoints on the GPU's Ldet."""
    w, h = 400, 300
    img = kaze_inputs.synth_image(w, h, 99)
    sg, _, st = O.schedule(5, 4, 1.6)
    assert st.max() > 32
    kz = make(w, h, octaves=5, sublevels=4, k_override=0.04)
    kz.batch = 1
    K.kaze_build_scale_space(kz.ctx, torch.from_numpy(img).cuda()[None])
    lv, _, _ = O.scale_space(img, octaves=5, sublevels=4, k_override=0.04)
    kps, counts, _ = _hessian_stage_isolated(O, kz, (0,), [lv], st, 20)
    Ld = gpu_levels(kz, 20, K.PLANE_LDET)
    kref, nref = O.extrema(Ld, 4, sg)
    got = K.Kaze.keypoints_numpy(kps, counts)[0]
    frac, _ = match_keypoints(kref, got, tol=1e-3)
    assert nref > 0 and int(counts[0]) == nref and frac >= 0.995
    kz.close()


# ------------------------------------------------------------------------------------------- prefilter, g1
@pytest.mark.parametrize("sigma0", [1.2, 2.5])
@pytest.mark.parametrize("w,h", [(333, 257), (640, 480)])
def test_generic_prefilter_levels(O, sigma0, w, h):
    """σ0 != 1.6 runs the generic separable prefilter k_prefilter<R> (R = 4, 8): level 0 within 2e-6 and every level
    within 1e-4 of the oracle (k injected); the device k lands in the oracle's bin."""
    img, ref = oracle_run(O, w, h, sigma0=sigma0)
    kz = make(w, h, sigma0=sigma0, k_override=ref["k"])
    K.kaze_build_scale_space(kz.ctx, torch.from_numpy(img).cuda()[None])
    lv = gpu_levels(kz, 16)
    assert rel_err(lv[0], ref["levels"][0]) < 2e-6
    for i in range(16):
        assert rel_err(lv[i], ref["levels"][i]) <= 1e-4, (i, rel_err(lv[i], ref["levels"][i]))
    kz.close()
    kz = make(w, h, sigma0=sigma0)
    K.kaze_build_scale_space(kz.ctx, torch.from_numpy(img).cuda()[None])
    k, _ = K.kaze_get_k(kz.ctx, 1)
    assert abs(k[0] / ref["k"] - 1) < 1e-5
    kz.close()


def test_g1_diffusivity_levels_and_conductivity(O):
    """diffusivity 1 (Eq. 3 g1 = exp(−|∇|²/k²)): every level within 1e-4 of the oracle (k injected) and
    the conductivity plane of the last step within 2e-5."""
    img, ref = oracle_run(O, 333, 257, octaves=3, sublevels=4, diffusivity=1)
    kz = make(333, 257, octaves=3, sublevels=4, k_override=ref["k"], diffusivity=1)
    K.kaze_build_scale_space(kz.ctx, torch.from_numpy(img).cuda()[None])
    lv = gpu_levels(kz, 12)
    for i in range(12):
        assert rel_err(lv[i], ref["levels"][i]) <= 1e-4, (i, rel_err(lv[i], ref["levels"][i]))
    c = torch.empty((257, 333), device="cuda")
    K.kaze_get_level(kz.ctx, 0, 0, K.PLANE_COND, c)
    cref = O.conductivity(ref["levels"][-2], ref["k"], 1)
    assert np.max(np.abs(c.cpu().numpy() - cref)) < 2e-5
    kz.close()


def test_g1_diffusivity_end_to_end(O):
    img, ref = oracle_run(O, 640, 480, diffusivity=1)
    kz = make(640, 480, diffusivity=1)
    kps, counts, desc = kz.extract(torch.from_numpy(img).cuda()[None])
    got = K.Kaze.keypoints_numpy(kps, counts)[0]
    assert ref["count"] > 0
    f1, idx = match_keypoints(ref["kps"], got)
    f2, _ = match_keypoints(got, ref["kps"])
    assert f1 >= 0.99 and f2 >= 0.99, (f1, f2, ref["count"], int(counts[0]))
    d = desc[0, : len(got)].cpu().numpy().astype(np.float64)
    m = idx >= 0
    a, b = ref["desc"][m], d[idx[m]]
    cos = np.sum(a * b, 1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1) + 1e-30)
    assert np.mean(cos >= 0.999) >= 0.99, np.mean(cos >= 0.999)
    kz.close()


# ------------------------------------------------------------------------------------------- graphs, edge cases
def test_graph_replay_across_sizes_AABBBA():
    """A graph bakes its size's texture table: replaying size A after size B was built and captured must still give
    the direct-launch result (one table per size, never rewritten while a graph uses it)."""
    A = torch.from_numpy(kaze_inputs.synth_batch(2, 333, 257)).cuda()
    B = torch.from_numpy(kaze_inputs.synth_batch(2, 300, 200, first=5)).cuda()
    g = make(333, 257, batch=2, octaves=3, sublevels=3, max_keypoints=4096)
    d = make(333, 257, batch=2, octaves=3, sublevels=3, max_keypoints=4096, flags=K.FLAG_NO_GRAPHS)
    refA, refB = d.extract(A), d.extract(B)
    oA, oB = g.alloc_outputs(2), g.alloc_outputs(2)
    for it, (img, o, ref) in enumerate([(A, oA, refA), (A, oA, refA), (B, oB, refB), (B, oB, refB), (B, oB, refB),
                                        (A, oA, refA), (A, oA, refA), (B, oB, refB)]):
        for t in o:
            t.zero_()
        K.kaze_extract(g.ctx, img, *o)
        torch.cuda.synchronize()
        for a, b in zip(o, ref):
            assert torch.equal(a, b), it
    g.close()
    d.close()


def test_describe_keypoints_on_levels_without_derivatives_are_zero():
    """Levels 0 and N−1 keep no (Lx, Ly) by default and levels outside 0..N−1 do not exist: such keypoints get a
    zero descriptor, angle 0 and flags = 1 instead of sampling stale or foreign memory."""
    w, h = 200, 150
    kz = make(w, h, octaves=3, sublevels=3, max_keypoints=64)
    img = torch.from_numpy(kaze_inputs.synth_image(w, h)).cuda()[None]
    kps, counts, desc = kz.extract(img)
    n = int(counts[0])
    assert n > 4
    arr = kps[0].cpu().numpy().view(K.KP_DTYPE).reshape(-1).copy()
    for j, lvl in enumerate([0, 8, -1, 9]):
        arr["level"][j] = lvl
        arr["angle"][j] = 1.0
    kk = torch.from_numpy(arr.view(np.int32).reshape(1, 64, 8).copy()).cuda()
    dd = torch.full((1, 64, 64), 7.0, device="cuda")
    K.kaze_describe(kz.ctx, kk, counts, dd)
    got = kk[0].cpu().numpy().view(K.KP_DTYPE).reshape(-1)
    assert torch.all(dd[0, :4] == 0) and np.all(got["flags"][:4] == 1) and np.all(got["angle"][:4] == 0)
    assert torch.equal(dd[0, 4:min(n, 64)], desc[0, 4:min(n, 64)])  # the others are untouched by the change
    kz.close()


def test_rot90_equivariance_on_the_gpu():
    """P13 on the device: the rotated image's keypoints are the rotated keypoints (x' = y, y' = W−1−x; >= 99% within
    0.05 px away from the border), their angles are θ − π/2 (48 windows) within 1e-3 rad for >= 99%, and their
    descriptors agree (cos >= 0.999 for >= 99%).  The column and row AOS passes swap roles under the rotation, so
    this also cross-checks the two solvers against each other."""
    img = kaze_inputs.synth_image(480, 360, 17)
    H, W = img.shape
    ka_ = make(W, H, ori_windows=48)
    kb_ = make(H, W, ori_windows=48)
    ra = ka_.extract(torch.from_numpy(img).cuda()[None])
    rb = kb_.extract(torch.from_numpy(np.ascontiguousarray(np.rot90(img))).cuda()[None])
    ka = K.Kaze.keypoints_numpy(ra[0], ra[1])[0]
    kb = K.Kaze.keypoints_numpy(rb[0], rb[1])[0]
    s = np.maximum(1, np.floor(1.6 * 2.0 ** (ka["level"] / 4.0) + 0.5))
    inner = np.minimum(np.minimum(ka["x"], ka["y"]), np.minimum(W - 1 - ka["x"], H - 1 - ka["y"])) >= 2 * s + 1
    ka_in = ka[inner]
    mapped = ka_in.copy()
    mapped["x"], mapped["y"] = ka_in["y"], W - 1 - ka_in["x"]
    frac, idx = match_keypoints(mapped, kb, tol=0.05)
    assert frac >= 0.99, frac
    m = idx >= 0
    dang = np.abs((kb["angle"][idx[m]] - (ka_in["angle"][m] - math.pi / 2) + math.pi) % (2 * math.pi) - math.pi)
    assert np.mean(dang < 1e-3) >= 0.99
    da = ra[2][0, : len(ka)].cpu().numpy()[inner][m].astype(np.float64)
    db = rb[2][0, : len(kb)].cpu().numpy()[idx[m]].astype(np.float64)
    cos = np.sum(da * db, 1) / (np.linalg.norm(da, axis=1) * np.linalg.norm(db, axis=1) + 1e-30)
    assert np.mean(cos >= 0.999) >= 0.99, np.mean(cos >= 0.999)
    ka_.close()
    kb_.close()


def test_overlapped_chunks_equal_sequential_chunks(tmp_path):
    """kaze_extract / kaze_extract_host with several chunks overlap each chunk's describe with the next chunk's
    build on a second stream (KAZE_OVERLAP, read once per process): the outputs equal those of a process that runs
    the chunks one after the other, bit for bit, direct and graph-replayed."""
    import os
    import subprocess
    import sys

    imgs = kaze_inputs.synth_batch(5, 200, 150, first=11)
    np.save(tmp_path / "imgs.npy", imgs)
    script = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "import paper_1706_06750_b200 as K\n"
        f"imgs = torch.from_numpy(np.load({str(tmp_path / 'imgs.npy')!r})).cuda()\n"
        "kz = K.Kaze(200, 150, batch=2, octaves=3, sublevels=3, max_keypoints=2048)\n"
        "out = kz.alloc_outputs(5)\n"
        "for _ in range(3): K.kaze_extract(kz.ctx, imgs, *out)\n"
        "torch.cuda.synchronize()\n"
        f"np.savez({str(tmp_path / 'seq.npz')!r}, *[t.cpu().numpy() for t in out])\n"
    )
    env = dict(os.environ, KAZE_OVERLAP="0")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    seq = np.load(tmp_path / "seq.npz")
    kz = make(200, 150, batch=2, octaves=3, sublevels=3, max_keypoints=2048)
    out = kz.alloc_outputs(5)
    dimg = torch.from_numpy(imgs).cuda()
    for it in range(3):  # direct, captured, replayed
        K.kaze_extract(kz.ctx, dimg, *out)
        torch.cuda.synchronize()
        for a, key in zip(out, ("arr_0", "arr_1", "arr_2")):
            assert np.array_equal(a.cpu().numpy(), seq[key]), (it, key)
    hk = np.zeros((5, 2048, 8), np.int32)
    hc = np.zeros(5, np.int32)
    hd = np.zeros((5, 2048, 64), np.float32)
    for it in range(3):
        K.kaze_extract_host(kz.ctx, np.ascontiguousarray(imgs), hk, hc, hd)
        assert np.array_equal(hc, seq["arr_1"])
        for i in range(5):
            n = int(hc[i])
            assert np.array_equal(hk[i, :n], seq["arr_0"][i, :n]) and np.array_equal(hd[i, :n], seq["arr_2"][i, :n])
    kz.close()


@pytest.mark.parametrize("knob", ["KAZE_ALTERNATE=0", "KAZE_HESS_FUSED=0", "KAZE_COND_TMA=0", "KAZE_COLS_PERSIST=0"])
def test_launch_order_and_hessian_form_do_not_change_results(tmp_path, knob):
    """Bit-identical outputs across launch-shape knobs (read once per process, so the reference runs in a
    subprocess): KAZE_ALTERNATE=0 runs every conductivity / AOS pass in ascending image order instead of alternating
    the order pass by pass; KAZE_HESS_FUSED=0 computes the Hessian with the two chain passes instead of the fused
    one (same operations, same order); KAZE_COND_TMA=0 loads every conductivity tile with global loads instead of
    staging the interior tiles with TMA tensor copies; KAZE_COLS_PERSIST=0 runs the AOS column pass one CTA per strip
    instead of persistent double-buffered CTAs."""
    import os
    import subprocess
    import sys

    w, h, n = 333, 257, 3
    imgs = kaze_inputs.synth_batch(n, w, h, first=21)
    np.save(tmp_path / "imgs.npy", imgs)
    script = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "import paper_1706_06750_b200 as K\n"
        f"imgs = torch.from_numpy(np.load({str(tmp_path / 'imgs.npy')!r})).cuda()\n"
        f"kz = K.Kaze({w}, {h}, batch={n}, max_keypoints=8192, flags=K.FLAG_ALL_DERIVATIVES)\n"
        f"out = kz.alloc_outputs({n})\n"
        "K.kaze_extract(kz.ctx, imgs, *out)\n"
        "torch.cuda.synchronize()\n"
        "lv = {}\n"
        f"for i in range({n}):\n"
        "    for p in (K.PLANE_LT, K.PLANE_LX, K.PLANE_LY, K.PLANE_LDET):\n"
        "        for l in range(16):\n"
        f"            t = torch.empty(({h}, {w}), device='cuda'); K.kaze_get_level(kz.ctx, i, l, p, t)\n"
        "            lv[f'{i}_{p}_{l}'] = t.cpu().numpy()\n"
        f"np.savez({str(tmp_path / 'ref.npz')!r}, *[t.cpu().numpy() for t in out], **lv)\n"
    )
    k, v = knob.split("=")
    r = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, **{k: v}), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = np.load(tmp_path / "ref.npz")
    kz = make(w, h, batch=n, max_keypoints=8192, flags=K.FLAG_ALL_DERIVATIVES)
    out = kz.alloc_outputs(n)
    K.kaze_extract(kz.ctx, torch.from_numpy(imgs).cuda(), *out)
    torch.cuda.synchronize()
    for a, key in zip(out, ("arr_0", "arr_1", "arr_2")):
        assert np.array_equal(a.cpu().numpy(), ref[key]), key
    for i in range(n):
        for p in (K.PLANE_LT, K.PLANE_LX, K.PLANE_LY, K.PLANE_LDET):
            lv = gpu_levels(kz, 16, p, img=i).astype(np.float32)
            for lvl in range(16):
                assert np.array_equal(lv[lvl], ref[f"{i}_{p}_{lvl}"]), (knob, i, p, lvl)
    kz.close()
