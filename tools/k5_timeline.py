"""K5 (assign_tc_kernel) event timeline of CTA 0 (run under gpurun; rebuilds libfms.so with -DK5_TIMELINE,
so run it on a scratch copy of the repo -- the gpurun box -- never before a measurement in the same call).

  python tools/k5_timeline.py [B=32]

Prints, per tile of CTA 0's range: producer x_empty wait, MMA d_empty / x_full waits and issue, and for the
lane-quarter-0 warp of the owning epilogue group: d_full wait, argmax (load + scan), stores.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FMS_NVCC_EXTRA"] = "-DK5_TIMELINE " + os.environ.get("K5_EXTRA", "")

import numpy as np
import torch

from paper_2007_14283_b200 import build as fbuild

fbuild.build(force=True)
import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
X = np.stack([synth.make_frame("C2", s).emb for s in range(B)])
pol = fms.default_policy(min_instance_px=min_instance_px(X.shape[1]), saturation_stop=1)
ctx = fms.Context(0)
ctx.set_option("graph", 0)
labels, centres, K, st = ctx.cluster(torch.from_numpy(X).cuda(), policy=pol, centres_cap=512)
torch.cuda.synchronize()
N = 6 * 1024 * 8
buf = (ctypes.c_longlong * N)()
lib = fms.lib()
lib.fms_k5_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.fms_k5_timeline(ctypes.addressof(buf), N) == N
h = np.frombuffer(buf, dtype=np.int64).reshape(6, 1024, 8)
t0 = h[1, 0, 0]
n_t = int((h[1, :, 3] > 0).sum())
print(f"B={B} K per frame {list(K[:8])}...  CTA 0 tiles {n_t}")
print("tile | prod x_empty wait | MMA: d_empty wait, x_full wait, issue | epi q0: d_full wait [ok at], argmax, stores")
for t in range(min(n_t, 64)):
    g = t % 4
    e = h[2 + g, t]
    print(f"{t:4d} | {h[0, t, 1] - h[0, t, 0]:6d} | {h[1, t, 1] - h[1, t, 0]:6d} {h[1, t, 2] - h[1, t, 1]:6d} "
          f"{h[1, t, 3] - h[1, t, 2]:6d} (start {h[1, t, 0] - t0:7d}) | {e[1] - e[0]:6d} [{e[1] - t0:7d}] "
          f"{e[2] - e[1]:6d} {e[3] - e[2]:6d}")
done = h[1, :n_t, 3]
print(f"MMA issue period over the range: {(done[n_t - 1] - done[0]) / max(n_t - 1, 1):.0f} cycles per tile")
