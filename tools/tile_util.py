"""Seed-row utilisation of K2's 128-row seed tiles on a C2 batch: active seed-iterations vs rows
computed (tiles x 128).  Usage: python tools/tile_util.py [config] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
frames = [synth.make_frame(cfg, i) for i in range(B)]
n, d = frames[0].n, frames[0].D
x = torch.from_numpy(np.stack([f.emb for f in frames])).cuda()
ctx = fms.Context(0)
ctx.set_option("profile_iter", 1)
pol = fms.default_policy(min_instance_px=min_instance_px(n), saturation_stop=1)
labels, centres, K, st = ctx.cluster(x, policy=pol, centres_cap=1024)
rs = st["run"]
n_chunks = (n + 2047) // 2048
tiles = rs["iter_items"] / n_chunks
print(dict(config=cfg, B=B, iter_launches=rs["iter_launches"], iter_ms=rs["iter_ms"], seed_iters=rs["iter_seed_iters"],
           tile_rows=tiles * 128, row_util=rs["iter_seed_iters"] / (tiles * 128),
           steps=rs["steps"], rounds=[f["rounds"] for f in st["frames"]][:8],
           round_K=[f["round_K"][:4] for f in st["frames"]][:4], round_iters=[f["round_iters"][:4] for f in st["frames"]][:4]))
