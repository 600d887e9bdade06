"""A small clustering run for compute-sanitizer (racecheck does not follow CUDA graphs with
conditional nodes, so the host-polled loop is used): C1 FIXED 64, S1sep OSOP, S32sep (DP = 32),
> 128 modes (the N = 256 assignment kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px

ctx = fms.Context(0)
ctx.set_option("graph", 0)
for cfg, kw in (("C1", dict(kind=0, n_seeds=64)), ("S1sep", {}), ("S32sep", {})):
    f = synth.make_frame(cfg, 0)
    pol = fms.default_policy(min_instance_px=min_instance_px(f.n), **kw)
    l, c, K, st = ctx.cluster(torch.from_numpy(f.emb).cuda(), policy=pol, centres_cap=512)
    print(cfg, K, st["status"], flush=True)
rng = np.random.default_rng(7)
dirs = []
while len(dirs) < 160:
    v = rng.standard_normal(16)
    v /= np.linalg.norm(v)
    if all(abs(float(v @ u)) < 0.7 for u in dirs):
        dirs.append(v)
x = np.concatenate([d + 0.04 * rng.standard_normal((40, 16)) for d in dirs]).astype(np.float32)
l, c, K, st = ctx.cluster(torch.from_numpy(x).cuda(), policy=fms.default_policy(has_background=0), centres_cap=512)
print("modes", K, st["status"])
