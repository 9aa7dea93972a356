"""Multi-GPU plumbing for the batch workload.

Images are independent units: rank r of P takes a contiguous shard of the batch and runs the whole path on
its own device with no data-path collective.  NCCL (torch.distributed) is used only to gather the per-image
keypoint counts (C1) and, optionally, the packed results (C2) — the method has no exchange step.

Collectives run on the tensors' device under NCCL; under gloo (CPU tests, or a one-GPU dry run of the multi-rank
bench with ``--dist-backend gloo``) they run on host copies, since gloo's all_gather does not take CUDA tensors.
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


def _host_collectives(group=None) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def _all_gather(out, inp, group=None):
    """all_gather_into_tensor on the tensors' device (NCCL) or through host copies (gloo)."""
    import torch.distributed as dist

    if _host_collectives(group) and inp.is_cuda:
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)
    return out


class CountGather:
    """C1 with the shard sizes settled once: ``gather(counts)`` is ONE all_gather_into_tensor of this rank's counts
    (padded to the largest shard) into a preallocated buffer, with no host synchronisation (NCCL) — the timed bench
    step calls it every step.  ``result()`` unpads (global image order); it reads the buffer, so it syncs."""

    def __init__(self, n_local: int, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.ws = dist.get_world_size(group)
        dev = torch.device("cpu") if device is None else torch.device(device)
        mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
        sizes = torch.empty(self.ws, dtype=torch.int64, device=dev)
        _all_gather(sizes, mine, group)
        self.sizes = [int(v) for v in sizes.cpu()]  # the one host sync, at set-up
        self.m = max(self.sizes) if self.sizes else 0
        self.n_local = n_local
        self.padded = torch.full((max(self.m, 1),), -1, dtype=torch.int32, device=dev)
        self.out = torch.empty(self.ws * max(self.m, 1), dtype=torch.int32, device=dev)

    def gather(self, counts):
        if counts.numel():
            self.padded[: counts.numel()].copy_(counts, non_blocking=True)
        return _all_gather(self.out, self.padded, self.group)

    def result(self):
        import torch

        m = max(self.m, 1)
        return torch.cat([self.out[r * m : r * m + self.sizes[r]] for r in range(self.ws)])


def gather_counts(counts, group=None):
    """C1: all-gather the per-image keypoint counts of every rank, in global image order.

    counts: 1-D int32 tensor (this rank's shard).  Shards may differ in length by one; they are padded to the
    longest, gathered with all_gather_into_tensor, and unpadded.  (One-shot form; the bench uses CountGather.)"""
    g = CountGather(counts.numel(), device=counts.device, group=None if group is None else group)
    g.gather(counts)
    return g.result()


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    dev = "cpu" if _host_collectives(group) else device
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(device=None, group=None):
    """dist.barrier that works for NCCL (device ids given) and gloo."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return
    if _host_collectives(group) or device is None:
        dist.barrier(group=group)
    else:
        dist.barrier(group=group, device_ids=[device.index if hasattr(device, "index") else int(device)])


def gather_results(kps, counts, desc, cap: int | None = None, group=None):
    """C2: every rank receives all ranks' keypoints and descriptors, truncated to their counts, in global image
    order (padded records gathered with all_gather_into_tensor over NCCL; the method itself needs no
    exchange, this is result collection).

    kps: [n_local, cap, 8] int32 (32-byte kaze_keypoint records), counts: [n_local] int32, desc: [n_local, cap, 64]
    float32, on this rank's device.  Each image's record block is padded to the largest count of any image of any
    rank, so one collective moves ws x n_max x m x 288 bytes.  Returns (list of [count_i, 8] int32 keypoint tensors,
    list of [count_i, 64] float32 descriptor tensors, global counts)."""
    import torch

    cap = kps.shape[1] if cap is None else cap
    cg = CountGather(counts.numel(), device=counts.device, group=group)
    cg.gather(counts)
    allc = cg.result().clamp(min=0, max=cap)
    ws, sizes, nmax = cg.ws, cg.sizes, max(cg.m, 1)
    m = max(1, int(allc.max()) if allc.numel() else 1)
    rec = torch.zeros((nmax, m, 72), dtype=torch.int32, device=kps.device)  # 8 keypoint words + 64 descriptor bits
    k = min(m, kps.shape[1])
    rec[: kps.shape[0], :k, :8] = kps[:, :k]
    rec[: desc.shape[0], :k, 8:] = desc[:, :k].contiguous().view(torch.int32)
    out = torch.empty((ws * nmax, m, 72), dtype=torch.int32, device=kps.device)
    _all_gather(out, rec, group)
    kl, dl = [], []
    g = 0
    for r in range(ws):
        for i in range(sizes[r]):
            c = int(allc[g])
            blk = out[r * nmax + i, :c]
            kl.append(blk[:, :8].contiguous())
            dl.append(blk[:, 8:].contiguous().view(torch.float32))
            g += 1
    return kl, dl, allc
