"""Host-side multi-GPU logic on CPU: sharding and the C1 count gather over gloo with world_size 2."""
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
