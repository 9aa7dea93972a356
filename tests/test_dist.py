"""Host-side multi-GPU logic on CPU: sharding, the C1 count gather and the C2 result gather over gloo, world size 2."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_06750_b200 import dist as D


@pytest.mark.parametrize("n,ws", [(256, 1), (256, 2), (256, 8), (255, 4), (3, 8), (0, 2)])
def test_shards_tile_the_batch(n, ws):
    covered = []
    for r in range(ws):
        f, c = D.shard(n, r, ws)
        covered.extend(range(f, f + c))
    assert covered == list(range(n))
    sizes = [D.shard(n, r, ws)[1] for r in range(ws)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    first, cnt = D.shard(n, rank, ws)
    local = torch.arange(first, first + cnt, dtype=torch.int32) * 10 + 7  # "counts" of this rank's images
    allc = D.gather_counts(local)
    mx = D.max_over_ranks(float(rank + 1))
    q.put((rank, allc.tolist(), mx))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [256, 5])
def test_gather_counts_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [i * 10 + 7 for i in range(n)]
    for rank, allc, mx in res:
        assert allc == want
        assert mx == 2.0


def _worker_results(rank, ws, port, n, cap, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    first, cnt = D.shard(n, rank, ws)
    g = torch.Generator().manual_seed(1000 + rank)
    counts = torch.tensor([(7 * (first + i)) % (cap + 3) for i in range(cnt)], dtype=torch.int32)  # some > cap
    kps = torch.randint(-1000, 1000, (cnt, cap, 8), dtype=torch.int32, generator=g)
    desc = torch.randn((cnt, cap, 64), generator=g)
    kl, dl, allc = D.gather_results(kps, counts, desc)
    q.put((rank, [t.tolist() for t in kl], [t.tolist() for t in dl], allc.tolist(),
           {first + i: (kps[i, : min(int(counts[i]), cap)].tolist(), desc[i, : min(int(counts[i]), cap)].tolist())
            for i in range(cnt)}))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [6, 3])
def test_gather_results_gloo_world2(n):
    """C2: every rank ends with every image's count-truncated keypoints and descriptors, bit for bit, in global
    image order, whatever the shard sizes (including a rank with fewer images) and counts above capacity."""
    cap = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_results, args=(r, 2, port, n, cap, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    truth = {}
    for r in res:
        truth.update(r[4])
    want_counts = [min((7 * i) % (cap + 3), cap) for i in range(n)]
    for rank, kl, dl, allc, _ in res:
        assert allc == want_counts
        assert len(kl) == n
        for i in range(n):
            assert kl[i] == truth[i][0] and dl[i] == truth[i][1]
