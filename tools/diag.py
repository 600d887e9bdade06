"""GPU diagnostic: run the CUDA path on small frames next to the oracle and print everything."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px
from tests.parity_util import ari, bijection, match_centres


def one(cfg, seed, **pol):
    f = synth.make_frame(cfg, seed)
    x = torch.from_numpy(f.emb).cuda()
    p = fms.default_policy(**pol)
    t = time.time()
    try:
        labels, centres, K, st = fms.cluster(x, policy=p, centres_cap=4096, allow=(5,))
    except Exception as e:
        print(cfg, seed, "GPU ERROR", e)
        return
    torch.cuda.synchronize()
    tg = time.time() - t
    base = dict(kind=1, n_seeds=128, gamma=0.9, L=2.0, H=8.0, P=0.99, has_background=1, min_instance_px=0,
                saturation_stop=0, max_rounds=8, rng_seed=0)
    base.update(pol)
    t = time.time()
    ro = oracle.cluster(f.emb, pol=oracle.policy(**base))
    to = time.time() - t
    lg = labels.cpu().numpy()[0]
    cg = centres.cpu().numpy()[0, :K[0]]
    fr = st["frames"][0]
    print(f"== {cfg} seed={seed} gpu {tg*1e3:.1f} ms  oracle {to*1e3:.0f} ms  K gpu={K[0]} orc={ro.K} "
          f"ari={ari(lg, ro.labels):.5f} bij={bijection(lg, ro.labels)}")
    if K[0] and ro.K:
        r, c, d = match_centres(cg, ro.centres)
        print(f"   centre cosdist max={d.max():.3e} mean={d.mean():.3e}")
    for k in ("rounds", "round_K", "round_iters", "round_conv", "round_Kc", "round_I", "round_cand", "seed_iters"):
        print(f"   {k:16s} gpu={fr[k]}  orc={ro.trace[k]}")


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0))
    one("C1", 0, kind=0, n_seeds=64)
    one("C1", 1, kind=0, n_seeds=64)
    f = synth.make_frame("S1sep", 0)
    one("S1sep", 0, n_seeds=16, min_instance_px=min_instance_px(f.n))
    one("S1", 0, min_instance_px=min_instance_px(f.n), saturation_stop=1)
    one("C2sep", 0, min_instance_px=200, saturation_stop=1)
    one("C2", 0, min_instance_px=200, saturation_stop=1)
    one("C2", 1, min_instance_px=200, saturation_stop=1)
