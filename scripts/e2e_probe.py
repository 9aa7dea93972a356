#!/usr/bin/env python
"""Where the end-to-end (host-buffer) path loses against the device path: times kaze_extract (device buffers) and
kaze_extract_host (pinned host buffers) on the bench workload, wall clock around each call after warm-up."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kaze_inputs  # noqa: E402
import paper_1706_06750_b200 as K  # noqa: E402

n, B = int(sys.argv[1]) if len(sys.argv) > 1 else 128, int(sys.argv[2]) if len(sys.argv) > 2 else 16
host = torch.from_numpy(kaze_inputs.synth_batch(n, 1920, 1200, distinct=4)).pin_memory()
dev = host.cuda()
kz = K.Kaze(1920, 1200, batch=B, max_keypoints=32768)
kps, cnt, desc = kz.alloc_outputs(n)
hk = torch.zeros((n, 32768, 8), dtype=torch.int32).pin_memory()
hc = torch.zeros(n, dtype=torch.int32).pin_memory()
hd = torch.zeros((n, 32768, 64), dtype=torch.float32).pin_memory()
for name, fn in [("device", lambda: K.kaze_extract(kz.ctx, dev, kps, cnt, desc)),
                 ("host", lambda: K.kaze_extract_host(kz.ctx, host, hk, hc, hd)),
                 ("host_nodesc", lambda: K.kaze_extract_host(kz.ctx, host, hk, hc, None))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {min(ts) * 1e3:.1f} ms for {n} images -> {n / min(ts):.0f} img/s", flush=True)
