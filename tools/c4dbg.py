import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth
from synth.frames import min_instance_px
import paper_2007_14283_b200 as fms
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fr = [synth.make_frame(cfg, 1000 + i) for i in range(B)]
x = torch.from_numpy(np.stack([f.emb for f in fr])).cuda()
pol = fms.default_policy(min_instance_px=min_instance_px(fr[0].n), saturation_stop=1)
t = time.time()
try:
    l, c, K, st = fms.cluster(x, policy=pol, centres_cap=4096)
    torch.cuda.synchronize()
    print("ok", K, time.time() - t, st["frames"][0])
except Exception as e:
    print("ERR", e)
