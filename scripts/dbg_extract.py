"""One small kaze_extract of two synthetic W x H images (for compute-sanitizer runs): python scripts/dbg_extract.py W H"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import kaze_inputs
import paper_1706_06750_b200 as K
w, h = int(sys.argv[1]), int(sys.argv[2])
imgs = kaze_inputs.synth_batch(2, w, h, first=5)
kz = K.Kaze(w, h, batch=2, octaves=4, sublevels=4, max_keypoints=8192)
out = kz.alloc_outputs(2)
K.kaze_extract(kz.ctx, torch.from_numpy(imgs).cuda(), *out)
torch.cuda.synchronize()
print("ok", out[1].cpu().numpy())
