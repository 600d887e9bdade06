"""Single-frame latency probe (run under gpurun, optionally under ncu): clusters one C2 frame a few
times through fms_cluster_batch (graph path) so an ncu launch list shows where a call's time goes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2007_14283_b200 as fms
import synth
from synth.frames import min_instance_px

f = synth.make_frame("C2", 0)
x = torch.from_numpy(f.emb[None]).cuda()
ctx = fms.Context(0)
if len(sys.argv) > 2:
    ctx.set_option("graph", int(sys.argv[2]))  # 0: host-polled loop (ncu does not see kernels in conditional graph nodes)
pol = fms.default_policy(min_instance_px=min_instance_px(x.shape[1]), saturation_stop=1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    labels, centres, K, st = ctx.cluster(x, policy=pol, centres_cap=256)
    e1.record()
    torch.cuda.synchronize()
    print(f"call {i}: {e0.elapsed_time(e1):.3f} ms, K={K[0]}, steps={st['run']['steps']}, launches={st['run']['launches']}")
