#!/usr/bin/env python
"""One kaze_match call at n = 65536 per side (random unit descriptors) for ncu (scripts/gpu_r02_*.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_06750_b200 as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
rng = np.random.default_rng(5)
X = rng.normal(size=(n, 64)).astype(np.float32)
X /= np.linalg.norm(X, axis=1, keepdims=True)
Y = rng.normal(size=(n, 64)).astype(np.float32)
Y /= np.linalg.norm(Y, axis=1, keepdims=True)
A, B = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
scratch = torch.empty(K.kaze_match_scratch_bytes(n, n), dtype=torch.uint8, device="cuda")
for _ in range(2):
    K.kaze_match(A, B, 0.8, scratch=scratch)
torch.cuda.synchronize()
print("done")
