"""Pins of the oracle's Euclidean metric (NEXT-4, reading R24: Eq. 4's distance with Eq. 3's flat
kernel on the raw embeddings).  CPU only.

  * library routine: with fixed seeds and gamma = 1 the method is the classic flat-kernel mean-shift
    that sklearn.cluster.MeanShift implements (radius-neighbour mean, stop below 1e-3 h, intensity =
    points within h of the mode, greedy suppression within h, nearest-centre labels): equal K, equal
    partition, centres within tol;
  * closed form: clusters tighter than h and farther apart than 2h converge in one update to the
    exact fp64 cluster mean;
  * invariance: a translation of the data translates the centres and keeps the labels (a cosine
    normalisation or renormalisation slipped into the Euclidean path breaks it).
"""
import numpy as np
import pytest

import oracle
from tests.parity_util import bijection, match_centres


def _blobs(k=5, per=60, d=6, spread=0.05, sep=3.0, seed=0, bg=0):
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((k, d)) * sep
    X = np.concatenate([C[j] + spread * rng.standard_normal((per, d)) for j in range(k)])
    truth = np.repeat(np.arange(k), per)
    p = rng.permutation(len(X))
    return X[p].astype(np.float32), truth[p], C


def _pol(**kw):
    base = dict(kind=oracle.SEEDS_FIXED, n_seeds=40, gamma=1.0, metric=oracle.METRIC_EUCLID, has_background=0)
    base.update(kw)
    return oracle.policy(**base)


@pytest.mark.parametrize("seed,h", [(0, 0.5), (1, 0.8), (2, 1.0)])
def test_matches_sklearn_meanshift(seed, h):
    from sklearn.cluster import MeanShift
    X, truth, _ = _blobs(seed=seed)
    pol = _pol(rng_seed=seed)
    r = oracle.cluster(X, h=h, pol=pol)
    assert r.status == 0
    # the same seeds: the oracle's selection (R11) re-run through its public select()
    idx = oracle.select(np.ones(len(X), np.uint8), 40, seed, 0)
    ms = MeanShift(bandwidth=h, seeds=X[idx].astype(np.float64), cluster_all=True, max_iter=300).fit(X)
    assert len(ms.cluster_centers_) == r.K
    assert bijection(r.labels, ms.labels_)
    cen = np.asarray(ms.cluster_centers_)
    D = np.linalg.norm(r.centres[:, None, :] - cen[None, :, :], axis=2)
    assert D.min(axis=1).max() <= 1e-3 * h


def test_tight_clusters_converge_to_exact_means():
    X, truth, _ = _blobs(k=4, per=50, d=5, spread=0.02, sep=4.0, seed=3)
    r = oracle.cluster(X, h=0.5, pol=_pol(n_seeds=20))
    assert r.status == 0 and r.K == 4
    assert bijection(r.labels, truth)
    means = np.stack([X[truth == j].astype(np.float64).mean(axis=0) for j in range(4)])
    D = np.linalg.norm(r.centres[:, None, :] - means[None, :, :], axis=2)
    assert D.min(axis=1).max() <= 1e-12


def test_translation_invariance():
    X, truth, _ = _blobs(k=3, per=80, d=4, spread=0.1, seed=4)
    t = np.array([5.0, -3.0, 0.25, 10.0], dtype=np.float32)
    r0 = oracle.cluster(X, h=0.6, pol=_pol(n_seeds=30))
    r1 = oracle.cluster(X + t, h=0.6, pol=_pol(n_seeds=30))
    assert r0.K == r1.K and np.array_equal(r0.labels, r1.labels)
    assert np.abs(r1.centres - r0.centres - t).max() <= 1e-5  # fp32 input rounding of X + t


def test_osop_recovers_blobs_and_zero_vectors_are_valid():
    X, truth, _ = _blobs(k=6, per=120, d=8, spread=0.05, sep=2.5, seed=5)
    X[0] = 0.0  # a zero embedding is an ordinary point under Eq. 4
    r = oracle.cluster(X, h=0.7, pol=_pol(kind=oracle.SEEDS_OSOP, n_seeds=8, gamma=0.9))
    assert r.status == 0
    assert r.K >= 6
    big = np.bincount(r.labels, minlength=r.K) > 1
    assert big.sum() == 6


def test_euclid_policy_validation():
    X, _, _ = _blobs()
    assert oracle.cluster(X, h=2.0, pol=_pol()).status == 0          # h >= 1 is fine for Eq. 4
    assert oracle.cluster(X, h=0.5, pol=_pol(profile=1)).status == oracle.E_INVALID
    assert oracle.cluster(X, h=0.5, pol=_pol(metric=3)).status == oracle.E_INVALID
