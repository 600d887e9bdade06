"""C5 (BASELINE configs[4]): a 92-frame 512x512 temporal stack clustered JOINTLY as one problem of
24.1M pixel embeddings (tracking-style: one cluster per cell track), on one B200.

The bench's frames/s metric is per 512x512 frame; here the unit is the stack: frames/s = 92 /
device time.  The whole stack fits one GPU (fp32 input 1.5 GB, limbs 0.77 GB), so pixel sharding
is not needed at this size.  --h takes a comma list: the C5 bandwidth sweep (BASELINE configs[4];
h = 0.05, 0.1, 0.2 in cosine distance, tol = h/1000).
Usage: python tools/c5_stack.py [--frames 92] [--h 0.05,0.1,0.2] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px


def ari(a, b):
    from math import comb
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    ct = np.zeros((ai.max() + 1, bi.max() + 1), dtype=np.int64)
    np.add.at(ct, (ai, bi), 1)
    s = sum(comb(int(v), 2) for v in ct.ravel() if v > 1)
    sa = sum(comb(int(v), 2) for v in ct.sum(1))
    sb = sum(comb(int(v), 2) for v in ct.sum(0))
    n2 = comb(len(a), 2)
    e = sa * sb / n2
    return (s - e) / (0.5 * (sa + sb) - e)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=92)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--h", default="0.1")
    args = ap.parse_args()
    t0 = time.time()
    emb, truth = synth.make_stack(args.frames, seed=0)
    gen_s = time.time() - t0
    n, d = emb.shape
    x = torch.from_numpy(emb).cuda()
    pol = fms.default_policy(min_instance_px=min_instance_px(512 * 512) * args.frames, saturation_stop=1)
    sub = np.random.default_rng(0).choice(n, size=min(n, 2_000_000), replace=False)
    out = []
    for h in [float(v) for v in args.h.split(",")]:
        fms.cluster(x, h=h, policy=pol, centres_cap=4096)
        times = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            labels, _, K, st = fms.cluster(x, h=h, policy=pol, centres_cap=4096)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        fr = st["frames"][0]
        res = dict(config="C5: %d x 512x512 stack, 16-D, 30 tracks, joint clustering" % args.frames, pixels=n,
                   h=h, ms=ms, frames_per_s=args.frames / (ms / 1e3), K=int(K[0]), rounds=fr["rounds"],
                   seeds=fr["seeds_total"], seed_iters=fr["seed_iters"],
                   ari_vs_truth_2M_sample=float(ari(labels[0].cpu().numpy()[sub], truth[sub])),
                   tflops_iter=fr["seed_iters"] * n * 4 * d / (ms / 1e3) / 1e12, gen_s=gen_s)
        print(json.dumps(res), flush=True)
        out.append(res)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out if len(out) > 1 else out[0], f, indent=1)


if __name__ == "__main__":
    main()
