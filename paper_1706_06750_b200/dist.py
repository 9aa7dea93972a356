"""Multi-GPU plumbing for the batch workload.

Images are independent units: rank r of P takes a contiguous shard of the batch and runs the whole path on
its own device with no data-path collective.  NCCL (torch.distributed) is used only to gather the per-image
keypoint counts (C1) and, optionally, the packed results (C2) — the method has no exchange step.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)))


def shard(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous, balanced shard of n units: (first, count).  Shards tile [0, n) exactly."""
    if world_size < 1 or not (0 <= rank < world_size) or n < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n, world_size)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def gather_counts(counts, group=None):
    """C1: all-gather the per-image keypoint counts of every rank, in global image order.

    counts: 1-D int32 tensor (this rank's shard).  Shards may differ in length by one; they are padded to the
    longest, gathered with all_gather_into_tensor, and unpadded."""
    import torch
    import torch.distributed as dist

    ws = dist.get_world_size(group)
    n_local = torch.tensor([counts.numel()], dtype=torch.int64, device=counts.device)
    sizes = torch.empty(ws, dtype=torch.int64, device=counts.device)
    dist.all_gather_into_tensor(sizes, n_local, group=group)
    m = int(sizes.max())
    padded = torch.full((m,), -1, dtype=counts.dtype, device=counts.device)
    padded[: counts.numel()] = counts
    out = torch.empty(ws * m, dtype=counts.dtype, device=counts.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    parts = [out[r * m : r * m + int(sizes[r])] for r in range(ws)]
    return torch.cat(parts)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_results(kps, counts, desc, cap: int | None = None, group=None):
    """C2: every rank receives all ranks' keypoints and descriptors, truncated to their counts, in global image
    order (padded records gathered with all_gather_into_tensor over NCCL; the method itself needs no
    exchange, this is result collection).

    kps: [n_local, cap, 8] int32 (32-byte kaze_keypoint records), counts: [n_local] int32, desc: [n_local, cap, 64]
    float32, on this rank's device.  Each image's record block is padded to the largest count of any image of any
    rank, so one collective moves ws x n_max x m x 288 bytes.  Returns (list of [count_i, 8] int32 keypoint tensors,
    list of [count_i, 64] float32 descriptor tensors, global counts)."""
    import torch
    import torch.distributed as dist

    ws = dist.get_world_size(group)
    cap = kps.shape[1] if cap is None else cap
    allc = gather_counts(counts, group).clamp(min=0, max=cap)
    n_local = torch.tensor([counts.numel()], dtype=torch.int64, device=counts.device)
    sizes = torch.empty(ws, dtype=torch.int64, device=counts.device)
    dist.all_gather_into_tensor(sizes, n_local, group=group)
    nmax = int(sizes.max())
    m = max(1, int(allc.max()) if allc.numel() else 1)
    rec = torch.zeros((nmax, m, 72), dtype=torch.int32, device=kps.device)  # 8 keypoint words + 64 descriptor bits
    k = min(m, kps.shape[1])
    rec[: kps.shape[0], :k, :8] = kps[:, :k]
    rec[: desc.shape[0], :k, 8:] = desc[:, :k].contiguous().view(torch.int32)
    out = torch.empty((ws * nmax, m, 72), dtype=torch.int32, device=kps.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    kl, dl = [], []
    g = 0
    for r in range(ws):
        for i in range(int(sizes[r])):
            c = int(allc[g])
            blk = out[r * nmax + i, :c]
            kl.append(blk[:, :8].contiguous())
            dl.append(blk[:, 8:].contiguous().view(torch.float32))
            g += 1
    return kl, dl, allc
