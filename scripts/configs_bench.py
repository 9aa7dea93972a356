#!/usr/bin/env python
"""Every BASELINE.json config on one B200, through the C ABI:

  C1  128x128, O = S = 2, scale space + Hessian detector only (kaze_build_scale_space + kaze_detect)
  C2  640x480, KAZE defaults, full path (kaze_extract)
  C3  1920x1200, full path incl. 64-D M-SURF (kaze_extract)
  C4  4096x4096 single image, full path (kaze_extract; the long AOS lines)
  C5  256 x 1920x1200 — bench.py's workload (see profiles/<round>/bench.json), repeated here at 16 images per launch

Single images: latency = median CUDA-event time of one call on the launching stream after warm-up (kaze_extract
replays the chunk as a CUDA graph once seen twice; the C1 stage pair launches directly with PDL).  Keypoint counts
are reported; parity of each config against the oracle lives in tests/ (test_gpu_parity.py).

usage: python scripts/configs_bench.py [--reps 20] [--out gpurun_out/configs]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kaze_inputs  # noqa: E402
import paper_1706_06750_b200 as K  # noqa: E402


def timed(fn, reps: int, warmup: int = 3) -> float:
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(warmup + reps):
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        if r >= warmup:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/configs")
    a = ap.parse_args()
    rows = []
    # C1: scale space + detector only
    img = torch.from_numpy(kaze_inputs.synth_image(128, 128)).cuda()[None]
    kz = K.Kaze(128, 128, batch=1, octaves=2, sublevels=2, max_keypoints=4096)
    kps, cnt, _ = kz.alloc_outputs(1)
    ms = timed(lambda: (K.kaze_build_scale_space(kz.ctx, img), K.kaze_detect(kz.ctx, kps, cnt)), a.reps)
    rows.append({"config": "C1 128x128 O=S=2 scale space + detector", "ms": ms, "img_s": 1e3 / ms,
                 "keypoints": int(cnt[0]), "launches": None})
    kz.close()
    # C2-C4: full path, one image per call
    for name, (W, H) in [("C2 640x480 full", (640, 480)), ("C3 1920x1200 full", (1920, 1200)),
                         ("C4 4096x4096 full", (4096, 4096))]:
        img = torch.from_numpy(kaze_inputs.synth_image(W, H)).cuda()[None]
        cap = 262144 if W * H > 1 << 22 else 65536
        kz = K.Kaze(W, H, batch=1, max_keypoints=cap)
        out = kz.alloc_outputs(1)
        ms = timed(lambda: K.kaze_extract(kz.ctx, img, *out), a.reps)
        rows.append({"config": name, "ms": ms, "img_s": 1e3 / ms, "keypoints": int(out[1][0]),
                     "memory_MiB": K.kaze_memory_footprint(kz.ctx)["total"] / 2**20})
        kz.close()
    # C5 slice: 16 images per launch, per-image throughput
    imgs = torch.from_numpy(kaze_inputs.synth_batch(32, 1920, 1200, distinct=4)).cuda()
    kz = K.Kaze(1920, 1200, batch=16, max_keypoints=32768)
    out = kz.alloc_outputs(32)
    ms = timed(lambda: K.kaze_extract(kz.ctx, imgs, *out), max(5, a.reps // 4))
    rows.append({"config": "C5 slice: 32 x 1920x1200, 16 per launch", "ms": ms, "img_s": 32e3 / ms,
                 "keypoints": float(out[1].float().mean())})
    kz.close()
    res = {"device": torch.cuda.get_device_name(0), "rows": rows}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    md = [f"# BASELINE configs on one {res['device']} (median CUDA-event time per call)", "",
          "| config | ms per call | images/s | keypoints (per image) |", "|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['config']} | {r['ms']:.3f} | {r['img_s']:.0f} | {r['keypoints']:.0f} |")
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
