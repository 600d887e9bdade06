"""The device-resident loop (include/fms.h option "graph", k_graph.cu): one CUDA graph launch per
call whose round and lockstep-step loops are WHILE conditional nodes must give exactly the results of
the host-polled loop (same kernels, same order of work per frame), with one host synchronisation per
call.  With option fuse_step = 1 the graph's step tail (K3 update,
ctl_step, the loop condition, the next plan) is one kernel (post_step_kernel, k_step.cu) whose CTAs
hand frames and the step over through completion counters; 12 C2 frames exercise that with many
frames in flight."""
import numpy as np
import pytest

import synth
from synth.frames import min_instance_px

pytestmark = pytest.mark.gpu


def _run(ctx, X, pol, cap=512, **kw):
    import torch
    labels, centres, K, st = ctx.cluster(torch.from_numpy(X).cuda(), policy=pol, centres_cap=cap, **kw)
    return labels.cpu().numpy(), centres.cpu().numpy(), K, st


@pytest.mark.parametrize("cfg,seeds,kind", [("S1", [0, 1, 2], 1), ("C1", [3], 0), ("S32sep", [0, 1], 1),
                                            ("C2", [4], 1), ("C2", list(range(10, 22)), 1)])
@pytest.mark.parametrize("fuse", [0, 1])
def test_graph_equals_host_loop(cfg, seeds, kind, fuse):
    import paper_2007_14283_b200 as fms
    X = np.stack([synth.make_frame(cfg, s).emb for s in seeds])
    n = X.shape[1]
    pol = (fms.default_policy(kind=0, n_seeds=64) if kind == 0 else
           fms.default_policy(min_instance_px=min_instance_px(n), saturation_stop=1))
    g = fms.Context(0)
    g.set_option("fuse_step", fuse)
    h = fms.Context(0)
    h.set_option("graph", 0)
    h.set_option("pdl", 0)  # the graph's step kernels use programmatic dependent launch; the reference does not
    lg, cg, Kg, sg = _run(g, X, pol)
    lh, ch, Kh, sh = _run(h, X, pol)
    assert Kg == Kh
    assert np.array_equal(lg, lh) and np.array_equal(cg, ch)
    assert [f for f in sg["frames"]] == [f for f in sh["frames"]]
    assert sg["run"]["host_syncs"] == 1 and sh["run"]["host_syncs"] > 1
    # a second call reuses the cached graph with other buffers
    lg2, cg2, Kg2, _ = _run(g, X[::-1].copy(), pol)
    assert Kg2 == Kg[::-1] and np.array_equal(lg2, lg[::-1])


def test_graph_euclid_and_host_entry_chunks():
    """Euclidean metric (NEXT-4) through the graph, and the host entry whose chunks of different sizes
    use several cached graphs."""
    import torch

    import paper_2007_14283_b200 as fms
    X = np.stack([synth.make_frame("S1", 20 + s).emb for s in range(5)])
    X = (X / np.linalg.norm(X, axis=-1, keepdims=True)).astype(np.float32)
    pol = fms.default_policy(min_instance_px=min_instance_px(X.shape[1]), saturation_stop=1)
    g, h = fms.Context(0), fms.Context(0)
    for c in (g, h):
        c.set_option("metric", 1)
        c.set_option("host_chunk", 2)
    h.set_option("graph", 0)
    lg, cg, Kg, _ = _run(g, X, pol, h=(0.2) ** 0.5)
    lh, ch, Kh, _ = _run(h, X, pol, h=(0.2) ** 0.5)
    assert Kg == Kh and np.array_equal(lg, lh) and np.array_equal(cg, ch)
    eh = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).pin_memory()
    for _ in range(2):
        lo = torch.full((5, X.shape[1]), -1, dtype=torch.int32).pin_memory()
        co = torch.zeros((5, 512, X.shape[2]), dtype=torch.float32).pin_memory()
        _, K, rs = g.cluster_host(eh, lo, co, 512, h=(0.2) ** 0.5, policy=pol)
        assert K == Kg and np.array_equal(lo.numpy(), lg) and np.array_equal(co.numpy(), cg)


def test_phase_times_profiled_loop():
    """fms_run_stats per-phase device times (option profile_iter, host-polled loop): every phase that
    ran has time, and the phases plus K2 account for the call's stream time."""
    import paper_2007_14283_b200 as fms
    X = np.stack([synth.make_frame("C2", s).emb for s in (30, 31, 32)])
    pol = fms.default_policy(min_instance_px=min_instance_px(X.shape[1]), saturation_stop=1)
    ctx = fms.Context(0)
    ctx.set_option("profile_iter", 1)
    _run(ctx, X, pol)  # warm-up (workspace, events)
    _, _, _, st = _run(ctx, X, pol)
    r = st["run"]
    for k in ("ms_prep", "ms_select", "ms_step_ctl", "ms_merge", "ms_assign", "iter_ms"):
        assert r[k] > 0, (k, r)
    parts = r["iter_ms"] + sum(r[k] for k in ("ms_prep", "ms_select", "ms_step_ctl", "ms_merge", "ms_assign",
                                              "ms_host_wait"))
    assert abs(parts - r["ms_total"]) <= 0.05 * r["ms_total"] + 0.05, (parts, r["ms_total"])
    assert r["iter_ms"] > r["ms_step_ctl"]
    # without profiling the graph path leaves them at zero
    ctx.set_option("profile_iter", 0)
    _, _, _, st = _run(ctx, X, pol)
    assert st["run"]["ms_select"] == 0 and st["run"]["host_syncs"] == 1
