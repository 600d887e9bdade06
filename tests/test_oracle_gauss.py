"""Pins of the oracle's Gaussian-profile iteration (NEXT-4, reading R23: w = exp(-(1 - x.s)/h), the
Gaussian profile of Eq. 2, on unit vectors).  CPU only.

Each pin is fixed by something other than the oracle's own formula:
  * symmetry: points placed symmetrically about an axis have their (unique) mode on the axis;
  * the h -> infinity limit: every weight -> 1, so one update gives the normalised global sum;
  * ascent: the update s' = normalize(grad F) of the convex KDE F(s) = sum exp(-(1 - x.s)/h) never
    decreases F (a wrong sign, a dropped weight or a missing term breaks it);
  * exact recovery of a well-separated generated frame (labels = ground truth up to a bijection).
"""
import numpy as np
import pytest

import oracle
import synth
from tests.parity_util import bijection


def _unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


@pytest.mark.parametrize("alpha,h", [(0.05, 0.1), (0.1, 0.1), (0.2, 0.3)])
def test_symmetric_ring_mode_is_the_axis(alpha, h):
    # 2 (D - 1) points at angle alpha from e_1, pairwise symmetric in every plane (e_1, e_k)
    D = 6
    pts = []
    for k in range(1, D):
        for sgn in (1.0, -1.0):
            v = np.zeros(D)
            v[0], v[k] = np.cos(alpha), sgn * np.sin(alpha)
            pts.append(v)
    x = _unit(pts)
    r = oracle.lockstep(x, x[:3], h, max_iter=300, tol=1e-13, gamma=1.0, profile=oracle.PROFILE_GAUSS)
    assert (r["status"] == 1).all()
    e1 = np.eye(D)[0]
    assert np.abs(r["seeds"] - e1).max() <= 1e-11


def test_two_points_mode_is_the_bisector():
    a = 0.07
    x = _unit([[np.cos(a), np.sin(a), 0.0], [np.cos(a), -np.sin(a), 0.0]])
    r = oracle.lockstep(x, x[:1], 0.1, max_iter=300, tol=1e-13, gamma=1.0, profile=oracle.PROFILE_GAUSS)
    assert r["status"][0] == 1
    assert np.abs(r["seeds"][0] - np.array([1.0, 0.0, 0.0])).max() <= 1e-11


def test_infinite_bandwidth_limit_is_the_mean_direction():
    rng = np.random.default_rng(3)
    x = _unit(rng.standard_normal((500, 8)))
    r = oracle.lockstep(x, x[:4], 1e9, max_iter=1, tol=1e-300, gamma=1.0, profile=oracle.PROFILE_GAUSS)
    m = _unit(x.sum(axis=0))
    for s in r["seeds"]:
        assert 1.0 - float(s @ m) <= 1e-12


def test_gaussian_update_ascends_the_kde():
    f = synth.make_frame("S1", 0)
    x = oracle.normalize(f.emb)
    h = 0.1
    F = lambda s: float(np.exp(-(1.0 - x @ s) / h).sum())  # noqa: E731  (Eq. 2 KDE, Gaussian profile)
    s = x[np.random.default_rng(1).choice(len(x), 12, replace=False)].copy()
    prev = np.array([F(v) for v in s])
    for _ in range(8):
        r = oracle.lockstep(x, s, h, max_iter=1, tol=1e-300, gamma=1.0, profile=oracle.PROFILE_GAUSS)
        s = r["seeds"]
        cur = np.array([F(v) for v in s])
        assert (cur >= prev - 1e-9 * prev).all()
        prev = cur


def test_gaussian_recovers_well_separated_frame():
    f = synth.make_frame("C1", 1)
    pol = oracle.policy(kind=oracle.SEEDS_FIXED, n_seeds=64, profile=oracle.PROFILE_GAUSS)
    r = oracle.cluster(f.emb, h=0.1, pol=pol)
    assert r.status == 0
    assert r.K == f.cells + 1
    assert bijection(r.labels, f.truth)


def test_profile_is_validated():
    f = synth.make_frame("C1", 0)
    r = oracle.cluster(f.emb, pol=oracle.policy(kind=oracle.SEEDS_FIXED, n_seeds=8, profile=7))
    assert r.status == oracle.E_INVALID
