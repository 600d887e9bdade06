"""Pins P8/P9 for the oracle's scalar pieces: Eq. 14/19 closed forms, SPEC worked values,
Monte-Carlo coverage, the gamma rule and the seed-selection key (CPU only)."""
import math

import mpmath
import numpy as np
import pytest

import oracle


def test_splitmix64_reference_sequence(golden):
    # R11 key generator == the public splitmix64 reference (state 0 sequence)
    g = golden["splitmix64_seed0_sequence"]["values"]
    golden_ratio = 0x9E3779B97F4A7C15
    for k, v in enumerate(g):
        assert oracle.lib().fmso_splitmix64((k * golden_ratio) % 2**64) == int(v, 16)


def test_key_is_bijective_per_round():
    # distinct pixels of one round never share a key (splitmix64 is a bijection of uint64)
    keys = {oracle.key(12345, 2, i) for i in range(20000)}
    assert len(keys) == 20000


@pytest.mark.parametrize("row", range(3))
def test_p_success_worked_values(golden, row):
    e = golden["p_success"][row]
    assert abs(oracle.p_success(e["N"], e["I"], e["r"]) - e["p"]) <= max(e["tol"], 1e-15)


@pytest.mark.parametrize("row", range(2))
def test_n_min_worked_values(golden, row):
    e = golden["n_min"][row]
    assert oracle.n_min(e["P"], e["I"], e["r"]) == e["N"]


def _p14_exact(N, I, r):
    mpmath.mp.dps = 50
    q = mpmath.mpf(r) / I
    return (1 - (1 - q) ** N) ** I


def test_n_min_is_exact_inversion_of_eq14():
    # SPEC S:293 / S:568: p(n_min) >= P and p(n_min - 1) < P on the whole grid, with Eq. 14
    # evaluated independently at 50 digits.
    for P in (0.9, 0.95, 0.99):
        for I in range(1, 21):
            for r in [x / 10 for x in range(1, 11)]:
                N = oracle.n_min(P, I, r)
                assert N >= 1
                assert _p14_exact(N, I, r) >= P - 1e-12, (P, I, r, N)
                if N > 1:
                    assert _p14_exact(N - 1, I, r) < P + 1e-12, (P, I, r, N)


def test_n_min_infinite_without_instances():
    assert oracle.n_min(0.99, 0, 0.5) == 2**63 - 1


def _coverage_exact(N, I, r):
    # exact probability that N uniform seeds hit each of I equal bins of total mass r
    # (inclusion-exclusion over the missed bins)
    return sum((-1) ** j * math.comb(I, j) * (1 - j * r / I) ** N for j in range(I + 1))


@pytest.mark.parametrize("N", [8, 16, 32, 64, 128])
def test_monte_carlo_coverage(N):
    # Eq. 14 is an independence approximation; Monte-Carlo must match the exact multinomial
    # coverage, and Eq. 14 is an upper bound of it.
    I, r, trials = 10, 1.0, 200000
    rng = np.random.default_rng(N)
    u = rng.random((trials, N))
    bins = np.minimum((u * I / r).astype(np.int64), I - 1)
    hit = np.zeros((trials, I), dtype=bool)
    np.put_along_axis(hit, bins, True, axis=1)
    freq = hit.all(axis=1).mean()
    ex = _coverage_exact(N, I, r)
    sd = math.sqrt(max(ex * (1 - ex), 1e-12) / trials)
    assert abs(freq - ex) <= 4 * sd + 1e-9
    assert oracle.p_success(N, I, r) >= ex - 1e-12
    if N >= 64:  # the two agree once coverage is likely (Fig. 9's operating point)
        assert abs(oracle.p_success(N, I, r) - ex) < 1e-3


def test_p_success_monotone():
    # strictly increasing in N, decreasing in I
    for I in (2, 5, 10):
        ps = [oracle.p_success(N, I, 0.5) for N in range(1, 200)]
        # strictly increasing until it saturates to 1.0 in fp64
        assert all(b > a or a > 1 - 1e-12 for a, b in zip(ps, ps[1:]))
        assert all(b >= a - 1e-15 for a, b in zip(ps, ps[1:]))
    assert oracle.p_success(64, 5, 0.5) > oracle.p_success(64, 10, 0.5)


def test_gamma_rule():
    L = oracle.lib()
    assert L.fmso_need(0.9, 10) == 9
    assert L.fmso_need(0.9, 128) == 116      # ceil(115.2)
    assert L.fmso_need(0.7, 10) == 7         # 0.7*10 = 7.000000000000001 in fp64
    assert L.fmso_need(1.0, 77) == 77


def test_select_is_k_smallest_keys_sorted_by_index():
    rng = np.random.default_rng(0)
    n = 5000
    cand = (rng.random(n) < 0.3).astype(np.uint8)
    for K in (1, 17, 128, 10000):
        out = oracle.select(cand, K, 99, 3)
        idx = np.nonzero(cand)[0]
        keys = np.array([oracle.key(99, 3, int(i)) for i in idx], dtype=np.uint64)
        want = np.sort(idx[np.argsort(keys, kind="stable")[:min(K, idx.size)]])
        assert np.array_equal(out, want)
        assert np.array_equal(out, oracle.select(cand, K, 99, 3))  # deterministic


def test_select_uniform_inclusion():
    # inclusion frequency over many salts is uniform (binomial, 4.5 sigma)
    n, K, salts = 64, 8, 4000
    cand = np.ones(n, dtype=np.uint8)
    cnt = np.zeros(n)
    for s in range(salts):
        cnt[oracle.select(cand, K, s, 0)] += 1
    p = K / n
    sd = math.sqrt(salts * p * (1 - p))
    assert np.all(np.abs(cnt - salts * p) <= 4.5 * sd)


@pytest.mark.parametrize("row", range(5))
def test_session_next_worked_values(golden, row):
    """O8 / NEXT-1 frame-to-frame seed count against SPEC's worked controller examples."""
    e = golden["session_next"][row]
    assert oracle.session_next(e["total"], e["nmin"], e["H"]) == e["N"]


def test_session_reaches_dead_band_on_a_stationary_sequence():
    """SPEC S:296 controller safety: with stationary (I, r) repeated updates stop changing once N is
    inside the dead band (N <= H N_min), and never go below N_min."""
    nmin, H = 100.0, 8.0
    N = 5000
    seen = [N]
    for _ in range(100):
        N = oracle.session_next(N, nmin, H)
        seen.append(N)
    assert seen[-1] == seen[-2] <= H * nmin and min(seen) >= nmin
