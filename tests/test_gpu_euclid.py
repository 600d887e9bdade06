"""NEXT-4 on the CUDA path: the Euclidean metric (fms_set_option "metric" = 1, reading R24: Eq. 4's
distance with the flat kernel on raw embeddings) against the fp64 oracle with the same metric (which
is pinned to sklearn's MeanShift).  Well-separated blobs: equal K, labels identical up to a bijection,
centres within 1e-4 h, identical per-round trace; d = 6 / 14 (one 16-lane operand row with the two
augmented columns) and 18 / 30 (32-lane rows)."""
import numpy as np
import pytest

import oracle
from tests.parity_util import bijection

pytestmark = pytest.mark.gpu


def _blobs(k, per, d, spread, sep, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((k, d)) * sep
    X = np.concatenate([C[j] + spread * rng.standard_normal((per, d)) for j in range(k)])
    return (X[rng.permutation(len(X))] * scale).astype(np.float32)


def _gpu(X, h, **pol):
    import torch
    import paper_2007_14283_b200 as fms
    ctx = fms.Context(0)
    ctx.set_option("metric", 1)
    labels, centres, K, st = ctx.cluster(torch.from_numpy(X).cuda(), h=h, policy=fms.default_policy(**pol),
                                         centres_cap=512)
    return labels.cpu().numpy()[0], centres.cpu().numpy()[0, :K[0]], K[0], st["frames"][0]


def _check(X, h, **pol):
    lg, cg, K, fr = _gpu(X, h, **pol)
    opol = dict(kind=1, n_seeds=128, gamma=0.9, has_background=1)
    opol.update(pol)
    ro = oracle.cluster(X, h=h, pol=oracle.policy(metric=oracle.METRIC_EUCLID, **opol))
    assert ro.status == 0
    assert K == ro.K, (K, ro.K, fr, ro.trace)
    assert bijection(lg, ro.labels)
    D = np.linalg.norm(cg[:, None, :].astype(np.float64) - ro.centres[None, :, :], axis=2)
    assert D.min(axis=1).max() <= 1e-4 * h
    for key in ("rounds", "round_K", "round_iters", "round_conv", "round_Kc"):
        assert fr[key] == ro.trace[key], key
    return K


@pytest.mark.parametrize("d,h,scale", [(6, 0.8, 1.0), (14, 1.0, 1.0), (18, 1.2, 1.0), (30, 1.5, 1.0),
                                       (6, 800.0, 1000.0), (6, 8e-4, 1e-3)])
def test_euclid_fixed_seeds_gamma1(d, h, scale):
    X = _blobs(6, 300, d, 0.08, 3.0, seed=d, scale=scale)
    _check(X, h, kind=0, n_seeds=48, gamma=1.0, has_background=0)


@pytest.mark.parametrize("seed", [0, 1])
def test_euclid_osop(seed):
    X = _blobs(8, 500, 10, 0.1, 3.0, seed=10 + seed)
    _check(X, 0.9, kind=1, n_seeds=16, gamma=0.9, has_background=0, rng_seed=seed)


def test_euclid_rejections():
    import paper_2007_14283_b200 as fms
    import torch
    ctx = fms.Context(0)
    ctx.set_option("metric", 1)
    x = torch.zeros((1, 100, 31), device="cuda")
    with pytest.raises(fms.FmsError):
        ctx.cluster(x, h=1.0)                       # d + 2 > 32
    ctx.set_option("kernel_profile", 1)
    with pytest.raises(fms.FmsError):
        ctx.cluster(torch.zeros((1, 100, 4), device="cuda"), h=1.0)
    with pytest.raises(fms.FmsError):
        ctx.set_option("metric", 5)


def test_huge_bandwidth_is_one_cluster():
    """a bandwidth hundreds of times the data scale used to overflow the fp16 threshold
    column (NaN similarities, every seed stalled).  h~ is clamped at 2 (scaled points are < 1 apart
    by 2), so every pixel is in every window: one cluster at the data mean, as in the oracle."""
    X = _blobs(3, 60, 6, 0.1, 2.0, seed=9)
    for h in (50.0, 1e6):
        lg, cg, K, fr = _gpu(X, h, kind=0, n_seeds=8, has_background=0)
        ro = oracle.cluster(X, h=h, pol=oracle.policy(kind=0, n_seeds=8, has_background=0,
                                                       metric=oracle.METRIC_EUCLID))
        assert ro.status == 0 and ro.K == 1 and K == 1
        assert np.all(lg == 0)
        assert np.abs(cg[0] - ro.centres[0]).max() <= 1e-4 * max(1.0, np.abs(ro.centres[0]).max())
