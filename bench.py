#!/usr/bin/env python
"""Benchmark of the B200-native KAZE hot path (BASELINE.json metric / configs[4]).

Workload: a batch of 256 synthetic 1920x1200 images, KAZE defaults (4 octaves x 4 sublevels, σ0 = 1.6, g2, k at
the 70th percentile), full path: nonlinear scale space (AOS) → Hessian detector → orientation + 64-D M-SURF.
The batch is sharded over the N ranks (strong scaling: 256 / N images per rank); a step is one pass of the whole
path over the rank's shard, plus the C1 all-gather of keypoint counts (NCCL) when N > 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kaze|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every key).  --impl reference times the fp64 CPU oracle
(oracle/, plain C) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KAZE ms/image @1920x1200; images/s at 1/2/4/8 B200; AOS % of HBM peak"
W_IMG, H_IMG, N_IMAGES = 1920, 1200, 256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kaze", choices=["kaze", "reference"])
    ap.add_argument("--images", type=int, default=N_IMAGES)
    ap.add_argument("--batch", type=int, default=32, help="images per launch (max_batch of the context); measured (r01) 1421/1536/1608/1651/1661/1627 img/s at 2/4/8/16/32/64, (r02, overlapped describe) 1703 at 16, 1719 at 32")
    ap.add_argument("--max-keypoints", type=int, default=32768)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--distinct", type=int, default=8, help="distinct generated images (the rest are shifts/flips)")
    ap.add_argument("--scheme", default="aos", choices=["aos", "fed"],
                    help="scale-space solver: AOS (Eq. 4, the north star) or FED cycles (Eq. 5, SURVEY 8 f1)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: a dry run of the multi-rank path, e.g. two ranks "
                         "sharing one GPU)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 8:
                continue
            for i, nm in enumerate(names):
                if r[4 + i].lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(n_local: int, first: int, distinct: int):
    import kaze_inputs

    return kaze_inputs.synth_batch(n_local, W_IMG, H_IMG, first=first, distinct=min(distinct, n_local))


def run_reference(args):
    """The oracle (plain fp64 C, OpenMP over images only) on the host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    import numpy as np

    import kaze_inputs
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    threads = max(1, cores)  # every host core the process may use (OpenMP over images, one image per thread)
    imgs = np.stack([kaze_inputs.synth_image(W_IMG, H_IMG, kaze_inputs.BASE_SEED + i) for i in range(threads)])
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        counts = oracle.run_batch(imgs, cap=1 << 17, nthreads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    sec = statistics.median(times)
    value = threads / sec
    cpu = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "configs[4]: 1920x1200 synthetic images, full KAZE path (bounded sample)",
                   "width": W_IMG, "height": H_IMG, "octaves": 4, "sublevels": 4},
        "ms_per_image": sec * 1e3 / threads,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "oracle",
                         "sample": f"{threads} images (seeds 1234..{1233 + threads}) per step, one per thread, "
                                   f"of the 1920x1200 full path; value from the median step of {len(times)}; "
                                   f"host '{cpu}', {cores} cores usable",
                         "keypoints": [int(c) for c in counts]},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_baseline_sample(host_imgs, runs: int = 3):
    """The oracle as it stands (OpenMP over images, one image per thread) on every usable host core: one image per
    core of the workload's own first images, median of `runs` runs — ~20-30 s of CPU work."""
    import numpy as np

    import oracle

    oracle.build()
    cores = max(1, len(os.sched_getaffinity(0)))
    k = min(cores, len(host_imgs))
    imgs = np.ascontiguousarray(host_imgs[:k])
    times = []
    for _ in range(runs):
        t0 = time.perf_counter()
        counts = oracle.run_batch(imgs, cap=1 << 17, nthreads=k)
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    return {"value": k / dt, "unit": "images/s", "cores": k, "kind": "oracle",
            "sample": f"{k} images of the workload (1920x1200, full path), one per thread on {k} of {cores} usable "
                      f"cores; median of {runs} runs: {dt:.2f} s per run ({', '.join(f'{t:.2f}' for t in times)}); "
                      f"{int(sum(counts))} keypoints"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1706_06750_b200 as K
    from paper_1706_06750_b200 import dist as D

    rank, local_rank, ws = D.world()
    # a gloo dry run may put several ranks on one visible GPU; NCCL runs one rank per GPU
    dev_index = local_rank % max(1, torch.cuda.device_count()) if args.dist_backend == "gloo" else local_rank
    dev = torch.device("cuda", dev_index)
    torch.cuda.set_device(dev)
    if ws > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    first, n_local = D.shard(args.images, rank, ws)
    assert args.warmup >= 3 or os.environ.get("KAZE_BENCH_ALLOW_SHORT"), "timing rules: W >= 3"

    host = make_inputs(n_local, first, args.distinct)  # untimed staging
    imgs = torch.from_numpy(host).to(dev)
    B = min(args.batch, max(1, n_local))
    scheme = K.SCHEME_FED if args.scheme == "fed" else K.SCHEME_AOS
    kz = K.Kaze(W_IMG, H_IMG, batch=B, device=dev_index, max_keypoints=args.max_keypoints, scheme=scheme)
    kps, counts, desc = kz.alloc_outputs(n_local)
    stream = torch.cuda.current_stream(dev)
    # C1's shard sizes are exchanged once here, outside the timed loop: a step's gather is then one collective
    # with no host sync
    cg = D.CountGather(n_local, device=dev) if ws > 1 else None

    def step():
        K.kaze_extract(kz.ctx, imgs, kps, counts, desc)
        if cg is not None:
            cg.gather(counts)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    D.barrier(dev)
    # Timed region: the production path (kaze_extract replays each chunk as a CUDA graph; profiling off).
    K.kaze_reset_profile(kz.ctx)  # also zeroes the launch counter
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize(dev)
        D.barrier(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        D.barrier(dev)
    ms_local = e0.elapsed_time(e1) / args.steps
    launches = K.kaze_launch_count(kz.ctx)
    # Per-kernel device times: the same K steps again with the context's CUDA events around every launch on its
    # stream (direct launches; this pass is not the headline and its step time is reported beside it).
    K.kaze_set_profiling(kz.ctx, True)
    K.kaze_reset_profile(kz.ctx)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize(dev)
    ms_profiled = p0.elapsed_time(p1) / args.steps
    prof = K.kaze_get_profile(kz.ctx)
    K.kaze_set_profiling(kz.ctx, False)
    ms = D.max_over_ranks(ms_local, device=dev)
    total_counts = cg.result() if cg is not None else counts
    kp_total = int(torch.clamp(total_counts, max=args.max_keypoints).sum())
    c2 = None
    if ws > 1:  # C2 once, untimed: every rank receives every image's records; check it against C1 and the local shard
        t0 = time.perf_counter()
        kl, dl, allc = D.gather_results(kps, counts, desc, cap=args.max_keypoints)
        torch.cuda.synchronize(dev)
        c2_ms = (time.perf_counter() - t0) * 1e3
        ok = len(kl) == args.images and bool(torch.equal(allc.cpu(), total_counts.cpu().clamp(0, args.max_keypoints)))
        for i in range(n_local):  # this rank's own images come back bit for bit
            c = min(int(counts[i]), args.max_keypoints)
            ok = ok and bool(torch.equal(kl[first + i].to(dev), kps[i, :c])) and bool(torch.equal(dl[first + i].to(dev), desc[i, :c]))
        ok = D.max_over_ranks(0.0 if ok else 1.0, device=dev) == 0.0
        c2 = {"ok": ok, "records": int(sum(t.shape[0] for t in kl)), "ms": c2_ms, "backend": args.dist_backend}

    # ---- roofline of the dominant kernel (largest device time in the step) ----
    peak, peak_kind = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    dname, d = dom
    achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9 if d["ms"] > 0 else 0.0
    aos_bytes = prof.get("aos_cols", {}).get("bytes", 0) + prof.get("aos_rows", {}).get("bytes", 0)
    aos_ms = prof.get("aos_cols", {}).get("ms", 0) + prof.get("aos_rows", {}).get("ms", 0)
    aos_gbs = aos_bytes / (aos_ms * 1e-3) / 1e9 if aos_ms > 0 else 0.0
    traffic = None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = summ.get("kernels", {}).get(dname, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "algo_bytes_per_launch": d["bytes"] / max(1, d["launches"]),
            "avg_launch_ms": d["ms"] / max(1, d["launches"]), "peak_source": peak_kind,
            "aos_achieved_gbs": aos_gbs, "aos_frac": aos_gbs / peak}
    step_kernel_ms = sum(v["ms"] for v in prof.values()) / args.steps

    # ---- end to end through the host-buffer C ABI (pinned host memory, copies inside the timed region) ----
    e2e = None
    if not args.no_e2e:
        h_imgs = torch.from_numpy(host).pin_memory()
        h_kps = torch.zeros((n_local, args.max_keypoints, 8), dtype=torch.int32).pin_memory()
        h_cnt = torch.zeros(n_local, dtype=torch.int32).pin_memory()
        h_desc = torch.zeros((n_local, args.max_keypoints, 64), dtype=torch.float32).pin_memory()
        K.kaze_extract_host(kz.ctx, h_imgs, h_kps, h_cnt, h_desc)  # warm-up
        torch.cuda.synchronize(dev)
        D.barrier(dev)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            K.kaze_extract_host(kz.ctx, h_imgs, h_kps, h_cnt, h_desc)
        torch.cuda.synchronize(dev)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e_ms = D.max_over_ranks(e2e_ms, device=dev)
        nk = int(torch.clamp(h_cnt, max=args.max_keypoints).sum())
        e2e = {"value": args.images / (e2e_ms * 1e-3), "unit": "images/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(n_local * H_IMG * W_IMG * 4),
               "d2h_bytes_per_step": int(n_local * 4 + nk * (32 + 256)),
               "api": "kaze_extract_host (pinned host buffers, chunked H2D/compute/D2H overlap)"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_sample(host)
        out = {
            "metric": METRIC,
            "value": args.images / (ms * 1e-3),
            "unit": "images/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "ms_per_image": ms / args.images * ws,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "configs[4]: batch of 256 synthetic 1920x1200 images sharded over the GPUs, "
                                   f"full path ({args.scheme.upper()} scale space, Hessian detector, orientation, "
                                   "64-D M-SURF)", "scheme": args.scheme,
                       "images": args.images, "width": W_IMG, "height": H_IMG, "octaves": 4, "sublevels": 4,
                       "max_batch": B, "max_keypoints": args.max_keypoints, "parallelism": f"dp{ws}",
                       "l2": "inputs (%.2f GB) larger than L2; no flush" % (args.images * H_IMG * W_IMG * 4 / 1e9),
                       "keypoints_per_image": kp_total / args.images},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * ws,
            "kernel_ms_per_step": step_kernel_ms,
            "ms_per_step_profiled": ms_profiled,
            "timing": "value: CUDA-graph replays of each step (the chunks' descriptor passes overlap the next chunk's scale space on a second stream), no per-kernel events; kernels/roofline: a second pass of the same steps, chunks one after the other, with CUDA events around every launch",
            "kernels": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                            "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] > 0 else None}
                        for k, v in prof.items()},
            "clocks": clocks.summary(),
        }
        if c2 is not None:
            out["c2_gather_results"] = c2
            out["config"]["dist_backend"] = args.dist_backend
            out["config"]["devices_visible"] = torch.cuda.device_count()
        if "describe" in prof and prof["describe"]["ms"] > 0:
            # gather roofline of the descriptor pass: 113 + 576 bilinear samples x 4 taps x 8 B
            # (float2 texels) = 22 KB per keypoint, served mostly by L1/L2 (each plane is read ~once from HBM)
            per_kp = (113 + 576) * 4 * 8
            kp_local = int(torch.clamp(counts, max=args.max_keypoints).sum())  # this rank's keypoints per step
            out["kernels"]["describe"]["gather_gbs"] = kp_local * per_kp * args.steps / (prof["describe"]["ms"] * 1e-3) / 1e9
            out["kernels"]["describe"]["gather_bytes_per_keypoint"] = per_kp
        print(json.dumps(out), flush=True)
    kz.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
