"""NEXT-3: the paper's simulation suite (Table 1) on the CUDA path.

1K..200K points x 18-D, 10 orthogonal/opposite clusters (synth.make_blobs), h = 0.1; the policy is
either Alg. 1 (every point a seed, FMS_SEEDS_ALL -- the exhaustive upper bound the paper's GPU_P
baseline corresponds to) or OSOP (Alg. 2 with the online seed optimisation).  Reports median
device time per frame over 5 runs (CUDA events) and checks K = 10 and labels = ground truth up to
a permutation.  The paper's numbers (Table 1, NVIDIA K80 via PyTorch; seconds per frame) are
printed beside ours for context only -- different hardware and a framework-level implementation.
Usage: python tools/table1.py [--out profiles/table1_r01.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2007_14283_b200 as fms
import synth

SIZES = [1000, 2000, 5000, 10000, 20000, 50000, 100000, 200000]
PAPER_OURS_S = [1.624, 1.618, 1.664, 1.698, 1.747, 1.892, 2.107, 2.692]   # Table 1 "Ours", s/frame (K80)
PAPER_GPU_P_S = [1.572, 1.559, 1.586, 1.594, 1.773, 2.256, 3.877, 7.561]  # Table 1 GPU_P (all points)


def bijective(a, b):
    pairs = set(zip(a.tolist(), b.tolist()))
    return len(pairs) == len(set(a.tolist())) == len(set(b.tolist()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    rows = []
    for i, n in enumerate(SIZES):
        emb, truth = synth.make_blobs(n, seed=0)
        x = torch.from_numpy(emb).cuda()
        pols = [("ALL (Alg. 1)", fms.default_policy(kind=fms.SEEDS_ALL)),
                ("OSOP (Alg. 2)", fms.default_policy(has_background=0))]
        for name, pol in pols:
            fms.cluster(x, policy=pol, centres_cap=64)
            times = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                labels, _, K, st = fms.cluster(x, policy=pol, centres_cap=64)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            ok = K[0] == 10 and bijective(labels[0].cpu().numpy(), truth)
            fr = st["frames"][0]
            rows.append(dict(n=n, policy=name, ms=float(np.median(times)), K=int(K[0]), truth_ok=bool(ok),
                             seeds=int(fr["seeds_total"]), seed_iters=int(fr["seed_iters"]),
                             paper_ours_s=PAPER_OURS_S[i], paper_gpu_p_s=PAPER_GPU_P_S[i]))
            print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
