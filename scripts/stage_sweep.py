#!/usr/bin/env python
"""Stage-timing sweep over the paper's image-size range + memory footprint.

The paper times CPU-KAZE and GPU-KAZE on "8 different image dimensions ranging from 240x400 to 1920x1200 with 6
images of varying complexity in each dimension" (Figs. 2-5), splits the time into the three
steps (scale space / detection / description, conclusion P:L465 "4:3:1"), and plots the GPU memory
footprint per size.  Only the endpoints (240x400, 480x640, 1200x1920) are named; the six sizes in
between are reading A26 of DESIGN.md.  The paper's image set is unavailable, so every image is the seeded
synthetic recipe at complexity c in {0.25, 0.5, 1, 1.5, 2, 3} (shapes and blobs per area x c).

Per size and image, on one B200 (cuda:0), through the C ABI calls a user makes:
  latency  — one image per call (max_batch = 1): kaze_build_scale_space, kaze_detect, kaze_describe timed apart
             with CUDA events on the launching stream, median of --reps after --warmup untimed runs;
  batched  — the same stages over a batch of --batch copies-with-shifts of the size's images per call (throughput
             mode of bench.py), per-image ms;
  memory   — kaze_memory_footprint of the max_batch = 1 context, and the cudaMemGetInfo drop around kaze_create.

usage: python scripts/stage_sweep.py [--out gpurun_out/stage_sweep] [--reps 20] [--warmup 3] [--batch 8]
Writes <out>.json and <out>.md.  Never run under a profiler for the numbers.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import kaze_inputs  # noqa: E402
import paper_1706_06750_b200 as K  # noqa: E402

# (width, height), landscape as BASELINE writes sizes; reading A26 (endpoints from P:L414, 480x640 from P:L439).
SIZES = [(400, 240), (640, 480), (800, 600), (1024, 768), (1280, 720), (1280, 960), (1600, 1000), (1920, 1200)]
COMPLEXITY = [0.25, 0.5, 1.0, 1.5, 2.0, 3.0]
STAGES = ("scale_space", "detect", "describe")


def _time_stages(kz: K.Kaze, imgs: torch.Tensor, reps: int, warmup: int) -> dict:
    n = imgs.shape[0]
    kps, counts, desc = kz.alloc_outputs(n)
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = {st: [] for st in STAGES}
    for r in range(warmup + reps):
        ev[0].record(s)
        K.kaze_build_scale_space(kz.ctx, imgs)
        ev[1].record(s)
        K.kaze_detect(kz.ctx, kps, counts)
        ev[2].record(s)
        K.kaze_describe(kz.ctx, kps, counts, desc)
        ev[3].record(s)
        torch.cuda.synchronize()
        if r >= warmup:
            for j, st in enumerate(STAGES):
                out[st].append(ev[j].elapsed_time(ev[j + 1]))
    med = {st: statistics.median(v) for st, v in out.items()}
    med["total"] = sum(med[st] for st in STAGES)
    med["keypoints"] = counts.cpu().numpy().astype(int).tolist()
    # the whole path through kaze_extract (one CUDA-graph replay per chunk once the chunk has been seen twice)
    g = []
    for r in range(warmup + reps):
        ev[0].record(s)
        K.kaze_extract(kz.ctx, imgs, kps, counts, desc)
        ev[1].record(s)
        torch.cuda.synchronize()
        if r >= max(warmup, 2):
            g.append(ev[0].elapsed_time(ev[1]))
    med["extract_graph"] = statistics.median(g)
    return med


def sweep(sizes, complexity, reps: int, warmup: int, batch: int) -> dict:
    torch.cuda.init()
    dev = torch.device("cuda", 0)
    rows = []
    for (W, H) in sizes:
        imgs = [kaze_inputs.synth_image(W, H, kaze_inputs.BASE_SEED + i, complexity=c) for i, c in enumerate(complexity)]
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        kz = K.Kaze(W, H, batch=1, max_keypoints=65536)
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        per_img = []
        for c, im in zip(complexity, imgs):
            t = _time_stages(kz, torch.from_numpy(im).to(dev)[None], reps, warmup)
            t["complexity"] = c
            t["keypoints"] = t["keypoints"][0]
            per_img.append(t)
        mem = K.kaze_memory_footprint(kz.ctx)  # after describe: texture table included
        kz.close()
        # throughput mode: `batch` images per call (the size's images, cycled)
        kb = K.Kaze(W, H, batch=batch, max_keypoints=65536)
        bimgs = torch.from_numpy(np.stack([imgs[i % len(imgs)] for i in range(batch)])).to(dev)
        tb = _time_stages(kb, bimgs, max(3, reps // 4), warmup)
        mem_b = K.kaze_memory_footprint(kb.ctx)
        kb.close()
        row = {
            "width": W, "height": H, "pixels": W * H,
            "latency_ms": {st: statistics.mean(t[st] for t in per_img) for st in (*STAGES, "total", "extract_graph")},
            "latency_ms_per_image": [{k: t[k] for k in (*STAGES, "total", "complexity", "keypoints")} for t in per_img],
            "keypoints_mean": statistics.mean(t["keypoints"] for t in per_img),
            "batched_ms_per_image": {st: tb[st] / batch for st in (*STAGES, "total", "extract_graph")},
            "batch": batch,
            "memory_bytes": mem,
            "memory_bytes_batch": mem_b,
            "cuda_free_drop_bytes": int(free0 - free1),
        }
        lat = row["latency_ms"]
        row["ratio_ss_det_desc"] = [lat[st] / lat["describe"] if lat["describe"] > 0 else None for st in STAGES]
        rows.append(row)
        print(f"{W}x{H}: latency {lat['total']:.3f} ms (ss {lat['scale_space']:.3f}, det {lat['detect']:.3f}, "
              f"desc {lat['describe']:.3f}), graph {lat['extract_graph']:.3f} ms, "
              f"batched {row['batched_ms_per_image']['extract_graph']:.3f} ms/img, "
              f"kps {row['keypoints_mean']:.0f}, mem {mem['total'] / 2**20:.1f} MiB", flush=True)
    return {
        "device": torch.cuda.get_device_name(0),
        "reading": "A26: sizes between the paper's endpoints chosen by us; complexity = shapes/blobs density factor",
        "reps": reps, "warmup": warmup, "rows": rows,
    }


def to_markdown(res: dict) -> str:
    L = [f"# Stage-timing sweep (SURVEY §8 f4) — {res['device']}", "",
         "Single-image latency through the C ABI (kaze_build_scale_space / kaze_detect / kaze_describe timed apart, "
         "direct launches, CUDA events, "
         f"median of {res['reps']} per image, mean over the 6 complexity levels); the whole path through kaze_extract "
         "(CUDA-graph replay) for one image and per image in batches of 8; keypoints; the context's device memory "
         "(kaze_memory_footprint, max_batch = 1).", "",
         "| size (WxH) | keypoints | scale space ms | detect ms | describe ms | total ms | ratio ss:det:desc | "
         "kaze_extract (graph) ms | batched ms/img (graph) | memory MiB (L_step scratch MiB) |",
         "|---|---|---|---|---|---|---|---|---|---|"]
    for r in res["rows"]:
        lat, m = r["latency_ms"], r["memory_bytes"]
        rat = ":".join(f"{x:.1f}" for x in r["ratio_ss_det_desc"])
        L.append(f"| {r['width']}x{r['height']} | {r['keypoints_mean']:.0f} | {lat['scale_space']:.3f} | "
                 f"{lat['detect']:.3f} | {lat['describe']:.3f} | {lat['total']:.3f} | {rat} | "
                 f"{lat['extract_graph']:.3f} | {r['batched_ms_per_image']['extract_graph']:.3f} | "
                 f"{m['total'] / 2**20:.1f} ({m['scratch'] / 2**20:.1f}) |")
    return "\n".join(L) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/stage_sweep")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--sizes", default="", help="comma list WxH (default: the 8-size ladder)")
    a = ap.parse_args()
    sizes = SIZES if not a.sizes else [tuple(int(v) for v in s.split("x")) for s in a.sizes.split(",")]
    res = sweep(sizes, COMPLEXITY, a.reps, a.warmup, a.batch)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write(to_markdown(res))


if __name__ == "__main__":
    main()
