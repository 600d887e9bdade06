"""NEXT-4 on the CUDA path: the Gaussian kernel profile (fms_set_option "kernel_profile" = 1, reading
R23: w = exp(-(1 - x.s)/h), Eq. 2) against the fp64 oracle with the same profile.

The weights are fp16 on the GPU (relative error ~2^-11, weights < 2^-24 flushed), so the bar is the
north_star's tolerance rather than bit-identity: on well-separated frames equal K, labels identical up
to a bijection and centres within 1e-4 cosine distance; on a soft-boundary frame ARI >= 0.999.
"""
import numpy as np
import pytest

import oracle
import synth
from synth.frames import min_instance_px
from tests.parity_util import bijection, match_centres

pytestmark = pytest.mark.gpu


def _ari(a, b):
    from math import comb
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    ct = np.zeros((ai.max() + 1, bi.max() + 1), dtype=np.int64)
    np.add.at(ct, (ai, bi), 1)
    s = sum(comb(int(v), 2) for v in ct.ravel() if v > 1)
    sa = sum(comb(int(v), 2) for v in ct.sum(1))
    sb = sum(comb(int(v), 2) for v in ct.sum(0))
    e = sa * sb / comb(len(a), 2)
    return (s - e) / (0.5 * (sa + sb) - e)


def _run(cfg, seed, fixed):
    import torch
    import paper_2007_14283_b200 as fms
    f = synth.make_frame(cfg, seed)
    kw = dict(kind=0, n_seeds=64) if fixed else dict(min_instance_px=min_instance_px(f.n), saturation_stop=1)
    ctx = fms.Context(0)
    ctx.set_option("kernel_profile", 1)
    labels, centres, K, st = ctx.cluster(torch.from_numpy(f.emb).cuda(), policy=fms.default_policy(**kw),
                                         centres_cap=1024)
    opol = oracle.policy(profile=oracle.PROFILE_GAUSS, **kw)
    ro = oracle.cluster(f.emb, h=0.1, pol=opol)
    assert ro.status == 0
    return f, labels.cpu().numpy()[0], centres.cpu().numpy()[0, :K[0]], K[0], ro


@pytest.mark.parametrize("cfg,seed,fixed", [("C1", 0, True), ("C1", 3, True), ("S1sep", 1, False),
                                            ("S32sep", 0, False)])
def test_gauss_well_separated_matches_oracle(cfg, seed, fixed):
    f, lg, cg, K, ro = _run(cfg, seed, fixed)
    assert K == ro.K
    assert bijection(lg, ro.labels)
    assert match_centres(cg, ro.centres)[2].max() <= 1e-4


def test_gauss_soft_frame_ari():
    f, lg, cg, K, ro = _run("S1", 0, False)
    assert _ari(lg, ro.labels) >= 0.999


def test_gauss_rejects_pixel_sharding_and_bad_values():
    import torch
    import paper_2007_14283_b200 as fms
    ctx = fms.Context(0)
    with pytest.raises(fms.FmsError):
        ctx.set_option("kernel_profile", 2)
    # the pixel-sharded exchange sums exact (integer-valued) flat-kernel window sums only
    f = synth.make_frame("C1", 0)
    ctx.set_option("kernel_profile", 1)
    ctx.set_pixel_shard(lambda buf, count, stream: 0, 0, 2, f.n, 0)
    x = torch.from_numpy(f.emb[: f.n // 2].copy()).cuda()
    with pytest.raises(fms.FmsError) as e:
        ctx.cluster(x, policy=fms.default_policy(kind=0, n_seeds=8), centres_cap=64)
    assert e.value.status == 2
