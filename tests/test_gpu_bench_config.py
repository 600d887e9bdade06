"""Parity in the launch configuration bench.py times (BASELINE configs[1], the metric config): one
fms_cluster_batch call over B = 96 resident C2 frames (512x512, 16-D, ~30 touching cells, full OSOP),
the first batch of bench.py's input pool.

At this size the oracle is checked on sampled outputs: two frames of the batch against the fp64
oracle (ARI >= 0.999, centres of the counted clusters within 1e-4 cosine distance), and eight frames
re-clustered alone on the GPU must be bit-identical to their slot in the batch (frames never
interact).  Every frame is checked for properties that hold at any size: status OK, labels in [0, K),
unit-norm centres.
"""
import numpy as np
import pytest

import oracle
import synth
from synth.frames import min_instance_px
from tests.parity_util import ari, match_centres

pytestmark = pytest.mark.gpu

B = 96


@pytest.fixture(scope="module")
def batch():
    import torch
    import paper_2007_14283_b200 as fms
    frames = [synth.make_frame("C2", i) for i in range(B)]  # bench.py's first input batch (rank 0)
    n, d = frames[0].n, frames[0].D
    X = torch.from_numpy(np.stack([f.emb for f in frames])).cuda()
    pol = fms.default_policy(min_instance_px=min_instance_px(n), saturation_stop=1)
    ctx = fms.Context(0)
    labels, centres, K, st = ctx.cluster(X, policy=pol, centres_cap=1024)
    torch.cuda.synchronize()
    return frames, X, pol, labels.cpu().numpy(), centres.cpu().numpy(), K, st


def test_every_frame_valid(batch):
    frames, X, pol, labels, centres, K, st = batch
    assert st["status"] == 0
    for b in range(B):
        k = K[b]
        assert st["frames"][b]["status"] == 0 and 1 <= k <= 1024
        lb = labels[b]
        assert lb.min() >= 0 and lb.max() < k
        assert np.abs(np.linalg.norm(centres[b, :k], axis=1) - 1.0).max() <= 1e-5


@pytest.mark.parametrize("b", [0, 57])
def test_sampled_frames_match_oracle(batch, b):
    frames, X, pol, labels, centres, K, st = batch
    f = frames[b]
    opol = oracle.policy(min_instance_px=min_instance_px(f.n), saturation_stop=1)
    ro = oracle.cluster(f.emb, h=0.1, pol=opol)
    assert ro.status == 0
    assert ari(labels[b], ro.labels) >= 0.999
    # the bench's FLOP basis: the run's own seed-iteration counts equal the oracle's
    fs = st["frames"][b]
    assert fs["seed_iters"] == ro.trace["seed_iters"]
    assert fs["round_seed_iters"] == ro.trace["round_seed_iters"]
    assert fs["round_K"] == ro.trace["round_K"] and fs["round_iters"] == ro.trace["round_iters"]
    big = np.nonzero(np.bincount(ro.labels, minlength=ro.K) >= min_instance_px(f.n))[0]
    assert match_centres(centres[b, :K[b]], ro.centres[big])[2].max() <= 1e-4


def test_sampled_frames_equal_single_runs(batch):
    import torch
    import paper_2007_14283_b200 as fms
    frames, X, pol, labels, centres, K, st = batch
    ctx = fms.Context(0)
    for b in [0, 1, 13, 31, 32, 64, 90, 95]:
        l1, c1, K1, _ = ctx.cluster(X[b], policy=pol, centres_cap=1024)
        assert K1[0] == K[b]
        assert np.array_equal(l1.cpu().numpy()[0], labels[b])
        assert np.array_equal(c1.cpu().numpy()[0], centres[b])
