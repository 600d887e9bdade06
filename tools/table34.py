"""NEXT-1: synthetic analogues of the paper's Table 3 (time per frame for N_initial = 64 / 128 / 256,
P:461-478) and Table 4 (H = 4 / 8 / 16) on B200.

For each ISBI-shaped cohort (P:451 frame sizes; BASELINE configs[2]) a 50-frame video (the paper
tested 50 frames per data set) of drifting cells whose track embeddings random-walk
(synth.make_stack with the cohort's size, cell count and radii) is clustered frame by frame through a
fms_session (include/fms.h: the OSOP seed count N carries from frame to frame).  Reported per
setting: mean device time per frame (CUDA events around each session step), mean seeds per frame and
over the first five frames, mean lockstep seed-iterations, mean K and the mean adjusted Rand index
against the generator's truth.  The paper's own numbers (K80, whole pipeline per frame) are carried
as context.

  python tools/table34.py [--frames 50] [--out profiles/table34_r02.json]
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
from synth.frames import CONFIGS, min_instance_px

PAPER_T3 = {"C3_hela": [2.59, 2.74, 2.98], "C3_gowt1": [12.18, 11.24, 11.26], "C3_simplus": [11.24, 11.72, 11.52],
            "C3_u373": [5.66, 5.64, 5.57]}
PAPER_T4 = {"C3_hela": [2.69, 2.74, 2.74], "C3_gowt1": [11.02, 11.24, 11.30], "C3_simplus": [11.36, 11.72, 11.81],
            "C3_u373": [5.56, 5.64, 5.67]}


def ari(a, b):
    from sklearn.metrics import adjusted_rand_score
    return float(adjusted_rand_score(a, b))


def run_session(frames, truth, n, n_init, H, ctx):
    pol = fms.default_policy(n_seeds=n_init, H=float(H), min_instance_px=min_instance_px(n), saturation_stop=1)
    sess = fms.Session(ctx, pol)
    ms, seeds, its, Ks, aris = [], [], [], [], []
    stream = torch.cuda.current_stream()
    for t, x in enumerate(frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        labels, centres, K, fs = sess.step(x, centres_cap=4096)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        seeds.append(fs["seeds_total"])
        its.append(fs["seed_iters"])
        Ks.append(K)
        aris.append(ari(labels.cpu().numpy(), truth[t]))
    sess.close()
    return {"ms_per_frame": float(np.mean(ms[1:])), "ms_first_frame": ms[0], "seeds_per_frame": float(np.mean(seeds)),
            "seeds_first5": float(np.mean(seeds[:5])), "seed_iters_per_frame": float(np.mean(its)),
            "K_mean": float(np.mean(Ks)), "ari_mean": float(np.mean(aris)), "ari_min": float(np.min(aris))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ctx = fms.Context(0)
    out = {"note": "synthetic cohort-shaped videos (synth.make_stack), GPU session per setting; paper values: "
                   "K80, whole pipeline, seconds per frame (context only)", "cohorts": {}}
    for cfg in ("C3_hela", "C3_gowt1", "C3_simplus", "C3_u373"):
        c = CONFIGS[cfg]
        emb, truth = synth.make_stack(a.frames, seed=7, H=c["H"], W=c["W"], D=c["D"], cells=c["cells"],
                                      radius=c["radius"])
        n = c["H"] * c["W"]
        frames = [torch.from_numpy(emb[t * n:(t + 1) * n]).cuda() for t in range(a.frames)]
        tr = [truth[t * n:(t + 1) * n] for t in range(a.frames)]
        res = {"frame": f"{c['H']}x{c['W']}x{c['D']}", "cells": c["cells"], "table3_N_initial": {}, "table4_H": {}}
        run_session(frames[:3], tr, n, 128, 8, ctx)  # warm-up (graph capture, workspace)
        for ni in (64, 128, 256):
            res["table3_N_initial"][str(ni)] = run_session(frames, tr, n, ni, 8, ctx)
        for H in (4, 8, 16):
            res["table4_H"][str(H)] = run_session(frames, tr, n, 128, H, ctx)
        res["paper_table3_s"] = dict(zip(["64", "128", "256"], PAPER_T3[cfg]))
        res["paper_table4_s"] = dict(zip(["4", "8", "16"], PAPER_T4[cfg]))
        out["cohorts"][cfg] = res
        print(cfg, json.dumps(res), flush=True)
        del frames
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
