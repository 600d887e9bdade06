import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_2007_14283_b200 as fms
from synth.frames import min_instance_px
B = 32
fr = [synth.make_frame("C2", 1000 + i) for i in range(B)]
x = torch.from_numpy(np.stack([f.emb for f in fr])).cuda()
n, d = fr[0].n, fr[0].D
lab = torch.empty((B, n), dtype=torch.int32, device="cuda"); cen = torch.empty((B, 1024, d), device="cuda")
ctx = fms.context(0); pol = fms.default_policy(min_instance_px=min_instance_px(n), saturation_stop=1)
st = torch.cuda.current_stream()
for poll in [int(a) for a in sys.argv[1:]]:
    ctx.set_option("poll_steps", poll)
    for _ in range(2): ctx.cluster_batch_ptr(x.data_ptr(), B, n, d, lab.data_ptr(), cen.data_ptr(), 1024, 0.1, 300, None, pol, st.cuda_stream)
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(8): rc, K, fs, rs = ctx.cluster_batch_ptr(x.data_ptr(), B, n, d, lab.data_ptr(), cen.data_ptr(), 1024, 0.1, 300, None, pol, st.cuda_stream)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    print(f"poll {poll}: {ms:.2f} ms/call, {B/ms*1e3:.0f} frames/s, launches {rs['launches']}, steps {rs['steps']}")
