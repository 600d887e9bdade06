"""Guard-pair statistic (option "guard_stats", fms_run_stats.guard_pairs): the lockstep
iteration pairs whose computed similarity lies within the certified error bound 2^-16 of tau = 1 - h
(Eq. 11) -- the window decisions the 3-term fp32 similarity cannot certify.  Pinned by brute
force: Alg. 1 (every pixel a seed) with a huge tolerance runs exactly one lockstep step over all
(pixel, pixel) pairs, so the count must equal the number of fp64 pixel-pair similarities in the band."""
import numpy as np
import pytest

import synth
from tests.test_gpu_parity import _dyadic_boundary_frame

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -16


def _run(X, h, guard, tol=None, **pol):
    import torch

    import paper_2007_14283_b200 as fms
    ctx = fms.Context(0)
    ctx.set_option("guard_stats", guard)
    x = torch.from_numpy(np.ascontiguousarray(X[None], dtype=np.float32)).cuda()
    labels, centres, K, st = ctx.cluster(x, h=h, tol=tol, policy=fms.default_policy(**pol), centres_cap=4096)
    torch.cuda.synchronize()
    return labels.cpu().numpy(), centres.cpu().numpy(), K, st


def test_guard_pairs_single_step_bruteforce():
    X = _dyadic_boundary_frame()
    h = 0.25
    _, _, _, st = _run(X, h, 1, tol=10.0, kind=2, gamma=1.0)
    fr = st["frames"][0]
    assert fr["round_iters"] == [1], fr["round_iters"]  # one lockstep step over every pixel as a seed
    xn = X.astype(np.float64) / np.linalg.norm(X.astype(np.float64), axis=1, keepdims=True)
    c = xn @ xn.T
    dist = np.abs(c - (1.0 - h))
    # no pair near the band's edge, where the GPU's ~1e-7 similarity error could move it across
    assert not np.any(np.abs(dist - EPS) < 1e-6)
    want = int(np.count_nonzero(dist < EPS))
    assert want > 0  # the ring and the rings at 0.75 -+ 2^-17 against e0 and each other
    assert st["run"]["guard_pairs"] == want, (st["run"]["guard_pairs"], want)


@pytest.mark.parametrize("cfg,pol", [("C1", dict(kind=0, n_seeds=64)), ("C2", dict(kind=1))])
def test_guard_kernel_results_unchanged(cfg, pol):
    """The counting instantiation computes exactly what the production one does."""
    f = synth.make_frame(cfg, 3)
    if cfg == "C2":
        from synth.frames import min_instance_px
        pol = dict(pol, min_instance_px=min_instance_px(f.n), saturation_stop=1)
    l0, c0, K0, s0 = _run(f.emb, 0.1, 0, **pol)
    l1, c1, K1, s1 = _run(f.emb, 0.1, 1, **pol)
    assert K0 == K1 and np.array_equal(l0, l1) and np.array_equal(c0, c1)
    assert s0["frames"] == s1["frames"]
    assert s0["run"]["guard_pairs"] == 0
    # a C2 frame (touching cells, noise) has pairs in the band; report the count per pair evaluated
    if cfg == "C2":
        pairs = s1["frames"][0]["seed_iters"] * f.n
        assert 0 < s1["run"]["guard_pairs"] < 1e-4 * pairs
