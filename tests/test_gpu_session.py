"""NEXT-1: frame sequences with the OSOP seed count carried across frames (O8) -- the CUDA
path's fms_session_* against the oracle's session on identical seeded frames."""
import numpy as np
import pytest

import oracle
import synth
from synth.frames import min_instance_px
from tests.parity_util import bijection, match_centres

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n_seeds", [("S1sep", 32), ("C2sep", 128)])
def test_session_matches_oracle_session(cfg, n_seeds):
    import torch
    import paper_2007_14283_b200 as fms
    frames = [synth.make_frame(cfg, s).emb for s in range(4)]
    mp = min_instance_px(frames[0].shape[0])
    ro, Ns = oracle.session(frames, pol=oracle.policy(n_seeds=n_seeds, min_instance_px=mp, saturation_stop=1))
    sess = fms.Session(fms.context(0), fms.default_policy(n_seeds=n_seeds, min_instance_px=mp, saturation_stop=1))
    for t, emb in enumerate(frames):
        assert sess.seeds == Ns[t]
        labels, centres, K, fs = sess.step(torch.from_numpy(emb).cuda(), centres_cap=1024)
        assert K == ro[t].K and fs["round_K"] == ro[t].trace["round_K"]
        assert bijection(labels.cpu().numpy(), ro[t].labels)
        _, _, dist = match_centres(centres[:K].cpu().numpy(), ro[t].centres)
        assert dist.max() <= 1e-4
    assert sess.seeds == oracle.session_next(ro[-1].trace["seeds_total"], ro[-1].trace["round_nmin"][-1], 8.0)


def test_session_reduction_branch_matches_oracle():
    """P:318 "if N is too large compared to N_min, N is reduced as N - N_min" (O8, R18): a session
    started with N = 4096 on 16K-pixel frames whose N_min is ~100 uses more than H * N_min seeds, so
    the next frame's N is reduced -- on the GPU exactly as in the oracle's session."""
    import torch
    import paper_2007_14283_b200 as fms
    frames = [synth.make_frame("S1sep", s).emb for s in range(4)]
    mp = min_instance_px(frames[0].shape[0])
    ro, Ns = oracle.session(frames, pol=oracle.policy(n_seeds=4096, min_instance_px=mp, saturation_stop=1))
    assert all(r.status == 0 for r in ro)
    t0 = ro[0].trace
    assert t0["seeds_total"] > 8.0 * t0["round_nmin"][-1] > 0          # the branch is taken
    assert Ns[1] == max(t0["seeds_total"] - int(t0["round_nmin"][-1]), int(t0["round_nmin"][-1]))
    sess = fms.Session(fms.context(0), fms.default_policy(n_seeds=4096, min_instance_px=mp, saturation_stop=1))
    for t, emb in enumerate(frames):
        assert sess.seeds == Ns[t]
        labels, centres, K, fs = sess.step(torch.from_numpy(emb).cuda(), centres_cap=1024)
        assert K == ro[t].K and fs["round_K"] == ro[t].trace["round_K"]
        assert fs["round_nmin"] == ro[t].trace["round_nmin"]
        assert bijection(labels.cpu().numpy(), ro[t].labels)
