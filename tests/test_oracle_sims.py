"""NEXT-3: the paper's simulation suite through the oracle (CPU only) -- the section 4.2.1 data sets of
Fig. 4 (circles, polarized with 8 and 4 clusters) and the Appendix A overlap frames
(P:533-541).  Pinned against what the paper and probability fix:

* seeding: with n_s seeds drawn without replacement (R11), every cluster is hit with the exact
  hypergeometric inclusion-exclusion probability; the oracle's success frequency over many salts
  must match it (3 sigma), and a run whose seeds hit every cluster recovers the truth exactly (P5);
* the polarized sets are SPEC's estimate_observation example: background 750 of 1500
  -> r = 0.5 exactly, I = #instances, and N_min = Eq. 19 at those values;
* Appendix A: no noise, so OSOP at P = 0.95 recovers the eight circles exactly and observes the
  generator's foreground ratio r; N_min is Eq. 19 at (0.95, 8, r).
"""
import math

import numpy as np
import pytest

import oracle
from synth.frames import make_circles, make_overlap, make_polarized


def _bijection(a, b):
    pairs = set(zip(a.tolist(), b.tolist()))
    return len(pairs) == len(set(a.tolist())) == len(set(b.tolist()))


def p_all_hit(sizes, n_seeds):
    """P(every cluster receives >= 1 of n_seeds distinct points drawn uniformly without replacement)
    by inclusion-exclusion over the clusters missed."""
    n = sum(sizes)
    k = len(sizes)
    total = math.comb(n, n_seeds)
    p = 0.0
    for mask in range(1 << k):
        miss = sum(sizes[j] for j in range(k) if mask >> j & 1)
        p += (-1) ** bin(mask).count("1") * math.comb(n - miss, n_seeds) / total
    return p


def test_circles_seed_success_rate_matches_hypergeometric():
    x, t = make_circles(0)
    sizes = np.bincount(t).tolist()
    p = p_all_hit(sizes, 64)
    assert 0.98 < p < 0.999                      # close to Eq. 14's 0.9883 (with replacement)
    runs, hits = 200, 0
    for s in range(runs):
        idx = oracle.select(np.ones(len(t), np.uint8), 64, s, 0)
        covered = len(set(t[idx].tolist())) == len(sizes)
        if s < 40:  # full clustering on a subset: a fully seeded run recovers the truth exactly
            r = oracle.cluster(x, h=0.1, pol=oracle.policy(kind=0, n_seeds=64, rng_seed=s, has_background=0))
            assert r.status == 0
            assert (r.K == 10 and _bijection(r.labels, t)) == covered
        hits += covered
    sd = math.sqrt(p * (1 - p) / runs)
    assert abs(hits / runs - p) <= 3 * sd + 1.0 / runs


@pytest.mark.parametrize("instances", [7, 3])
def test_polarized_sets_observation_and_recovery(instances):
    x, t = make_polarized(0, instances)
    assert np.bincount(t)[0] == 750 and len(t) == 1500
    r = oracle.cluster(x, h=0.1, pol=oracle.policy(n_seeds=64, rng_seed=2))
    assert r.status == 0 and r.K == instances + 1 and _bijection(r.labels, t)
    tr = r.trace
    assert tr["round_I"][-1] == instances and tr["round_r"][-1] == 0.5
    assert tr["round_nmin"][-1] == oracle.n_min(0.99, instances, 0.5)


@pytest.mark.parametrize("spacing", [300, 200, 150])
def test_appendix_a_overlap_frames(spacing):
    x, t = make_overlap(spacing)
    r_true = 1.0 - np.count_nonzero(t == 0) / t.size
    r = oracle.cluster(x, h=0.1, pol=oracle.policy(P=0.95, rng_seed=0))
    assert r.status == 0 and r.K == 9 and _bijection(r.labels, t)
    tr = r.trace
    assert tr["round_I"][-1] == 8 and tr["round_r"][-1] == r_true
    assert tr["round_nmin"][-1] == oracle.n_min(0.95, 8, r_true)
