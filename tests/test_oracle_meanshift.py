"""Pins P1-P7 for the oracle's mean-shift, merge and assignment (CPU only).

Each test checks the oracle against something the paper or mathematics fixes, not against a
re-typed copy of its own formula: fixed points (P1), monotone ascent of the flat-kernel density
(P2), non-empty windows (P3), closed-form centres and exact recovery on well-separated frames
(P4/P5), an independently written per-point Alg. 1 loop (P6), and sklearn's neighbour routines (P7).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
from sklearn.neighbors import NearestNeighbors

import oracle
import synth
from synth.frames import min_instance_px


def _unit(x):
    return x / np.linalg.norm(x, axis=-1, keepdims=True)


def _bijection(a, b):
    """labels a and b are the same partition (contingency table has one nonzero per row/col)."""
    pairs = set(zip(a.tolist(), b.tolist()))
    return len(pairs) == len(set(a.tolist())) == len(set(b.tolist()))


# --------------------------------------------------------------------------------------------
# geometry: Eq. 1/9 distance, Eq. 11 flat kernel (inclusive), normalisation
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("row", range(3))
def test_cosine_distance_worked(golden, row):
    e = golden["cosine_distance"][row]
    X = oracle.normalize(np.array([e["a"], e["b"]], dtype=np.float32))
    assert abs((1.0 - X[0] @ X[1]) - e["d"]) < 1e-15


@pytest.mark.parametrize("row", range(3))
def test_flat_kernel_worked(golden, row):
    # a point at cosine distance `dist` from the seed is in the window iff dist <= h (Eq. 11)
    e = golden["flat_kernel"][row]
    c = 1.0 - e["dist"]
    s = np.array([1.0, 0.0])
    x = np.array([[c, np.sqrt(max(0.0, 1 - c * c))]])
    g, cnt = oracle.window(x, s, e["h"])
    assert cnt == e["k"]


def test_window_boundary_is_inclusive_exactly():
    h = 0.25                                   # tau = 0.75 exactly representable
    s = np.array([1.0, 0.0, 0.0])
    x = np.array([[0.75, np.sqrt(1 - 0.75 ** 2), 0.0],
                  [np.nextafter(0.75, 0.0), np.sqrt(1 - 0.75 ** 2), 0.0]])
    g, cnt = oracle.window(x, s, h)
    assert cnt == 1 and g[0] == 0.75


def test_normalize_unit_and_zero_norm():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((100, 7)).astype(np.float32) * 5
    X = oracle.normalize(x)
    assert np.allclose(np.linalg.norm(X, axis=1), 1.0, atol=1e-15)
    bad = x.copy()
    bad[13] = 0
    with pytest.raises(ValueError):
        oracle.normalize(bad)
    r = oracle.cluster(bad, pol=oracle.policy(kind=oracle.SEEDS_FIXED, n_seeds=4))
    assert r.status == oracle.E_ZERO_NORM


def test_invalid_arguments():
    x = np.ones((10, 4), dtype=np.float32)
    assert oracle.cluster(x, h=0.0).status == oracle.E_INVALID
    assert oracle.cluster(x, h=1.0).status == oracle.E_INVALID
    assert oracle.cluster(x, pol=oracle.policy(max_rounds=0)).status == oracle.E_INVALID


def test_window_equals_sklearn_radius_neighbors():
    # P7: for unit vectors, 1 - x.y <= h  <=>  |x - y|_2 <= sqrt(2h)
    rng = np.random.default_rng(2)
    X = _unit(rng.standard_normal((3000, 6)))
    X[:1500] = _unit(X[:1500] * 0.1 + np.array([1, 0, 0, 0, 0, 0]))
    h = 0.1
    nn = NearestNeighbors(radius=np.sqrt(2 * h)).fit(X)
    for j in range(0, 3000, 97):
        s = X[j]
        g, cnt = oracle.window(X, s, h)
        ind = nn.radius_neighbors(s[None], return_distance=False)[0]
        dots = X @ s
        band = np.abs(dots - (1 - h)) < 1e-12      # ignore pairs within rounding of the boundary
        want = set(ind.tolist()) - set(np.nonzero(band)[0].tolist())
        got = set(np.nonzero(dots >= 1 - h)[0].tolist()) - set(np.nonzero(band)[0].tolist())
        assert got == want
        if not band.any():
            assert cnt == len(ind)
            assert np.allclose(g, X[np.sort(ind)].sum(0), atol=1e-9)


# --------------------------------------------------------------------------------------------
# mean-shift iteration: P1 fixed points, P2 monotone ascent, P3 non-empty windows
# --------------------------------------------------------------------------------------------

def _objective(X, s, tau):
    # flat-kernel density of Eq. 2 with R2 (spherical Epanechnikov profile): F(s) = sum max(0, x.s - tau)
    return np.maximum(0.0, X @ s - tau).sum()


@pytest.mark.parametrize("cfg", ["S1", "C1"])
def test_monotone_ascent_and_nonempty_windows(cfg):
    f = synth.make_frame(cfg, 3)
    X = oracle.normalize(f.emb)
    h = 0.1
    rng = np.random.default_rng(0)
    seeds = X[rng.choice(X.shape[0], 64, replace=False)].copy()
    for _ in range(25):
        F0 = np.array([_objective(X, s, 1 - h) for s in seeds])
        out = oracle.lockstep(X, seeds, h, max_iter=1, gamma=1.0)
        assert not np.any(out["status"] == 2)                     # P3: never stalled
        seeds = out["seeds"]
        assert all(oracle.window(X, s, h)[1] >= 1 for s in seeds)  # P3: next window non-empty
        F1 = np.array([_objective(X, s, 1 - h) for s in seeds])
        assert np.all(F1 >= F0 - 1e-9)                            # P2


@pytest.mark.parametrize("cfg", ["S1", "C1"])
def test_polish_mode_reaches_exact_fixed_points(cfg):
    # P1: with tol -> 0 every seed stops only when its window no longer changes; then the mode
    # reproduces itself: normalize(sum_{W(m)} x) == m.
    f = synth.make_frame(cfg, 4)
    X = oracle.normalize(f.emb)
    h = 0.1
    rng = np.random.default_rng(1)
    seeds = X[rng.choice(X.shape[0], 48, replace=False)].copy()
    out = oracle.lockstep(X, seeds, h, max_iter=300, tol=1e-300, gamma=1.0)
    conv = out["status"] == 1
    assert conv.mean() > 0.9
    for m in out["seeds"][conv]:
        g, cnt = oracle.window(X, m, h)
        assert np.linalg.norm(g / np.linalg.norm(g) - m) <= 1e-12


def _shift_to_mode(X, x0, tau, tol, max_iter):
    """Independent per-point Alg. 1 loop written with numpy primitives."""
    s = x0.copy()
    for t in range(1, max_iter + 1):
        m = (X @ s) >= tau
        g = X[m].sum(axis=0)
        s2 = g / np.linalg.norm(g)
        d = np.linalg.norm(s2 - s)
        s = s2
        if d < tol:
            return s, t, True
    return s, max_iter, False


def test_all_points_mode_reduces_to_alg1():
    # P6 / SPEC S:210: gamma = 1 with every point a seed is Alg. 1.
    rng = np.random.default_rng(5)
    cen = _unit(rng.standard_normal((4, 5)))
    X = np.concatenate([_unit(c + 0.08 * rng.standard_normal((120, 5))) for c in cen]
                       + [_unit(rng.standard_normal((40, 5)))])
    h, tol = 0.1, 1e-4
    out = oracle.lockstep(X, X, h, max_iter=300, tol=tol, gamma=1.0)
    for j in range(X.shape[0]):
        s, t, ok = _shift_to_mode(X, X[j], 1 - h, tol, 300)
        assert ok == (out["status"][j] == 1)
        assert np.linalg.norm(s - out["seeds"][j]) < 1e-9
        assert t == out["seed_iters_each"][j]


def test_early_stop_bound_and_status():
    f = synth.make_frame("S1", 0)
    X = oracle.normalize(f.emb)
    rng = np.random.default_rng(2)
    K = 100
    seeds = X[rng.choice(X.shape[0], K, replace=False)]
    out = oracle.lockstep(X, seeds, 0.1, gamma=0.9)
    st = out["status"]
    assert set(np.unique(st).tolist()) <= {1, 3}
    assert (st == 1).sum() >= 90                     # ceil(0.9 * 100)
    assert (st == 3).sum() <= int(np.ceil(0.1 * K))
    # converged modes are fixed points within tol
    for m in out["seeds"][st == 1]:
        g, _ = oracle.window(X, m, 0.1)
        assert np.linalg.norm(g / np.linalg.norm(g) - m) < 1e-4
    # intensity of a mode = number of points in its window (Eq. 2 density at the mode, R10),
    # pinned to sklearn's radius query (|x - m| <= sqrt(2h) for unit vectors)
    nn = NearestNeighbors(radius=np.sqrt(2 * 0.1)).fit(X)
    modes = out["seeds"][st == 1]
    got = out["intensity"][st == 1]
    want = np.array([len(r) for r in nn.radius_neighbors(modes, return_distance=False)])
    band = np.array([np.any(np.abs(X @ m - 0.9) < 1e-12) for m in modes])
    assert np.array_equal(got[~band], want[~band])


# --------------------------------------------------------------------------------------------
# merge (R10) and assignment (Alg. 2 l.12-14)
# --------------------------------------------------------------------------------------------

def test_merge_is_greedy_nms():
    # characterisation of greedy NMS in (intensity desc, origin asc) order: kept centres are
    # pairwise farther than rho, and every dropped mode lies within rho of a kept, higher-ranked one.
    rng = np.random.default_rng(7)
    base = _unit(rng.standard_normal((6, 8)))
    pool = _unit(np.repeat(base, 12, axis=0) + 0.12 * rng.standard_normal((72, 8)))
    inten = rng.integers(1, 40, size=72)
    origin = rng.permutation(1000)[:72]
    rho = 0.1
    keep = oracle.merge(pool, inten, origin, rho)
    rank = {j: r for r, j in enumerate(sorted(range(72), key=lambda j: (-inten[j], origin[j])))}
    kept = set(keep.tolist())
    assert [rank[j] for j in keep] == sorted(rank[j] for j in keep)   # kept in rank order
    for a in keep:
        for b in keep:
            if a != b:
                assert 1 - pool[a] @ pool[b] > rho
    for j in range(72):
        if j not in kept:
            assert any(1 - pool[j] @ pool[k] <= rho and rank[k] < rank[j] for k in kept)
    # idempotent, duplicates merge, far-apart survive
    keep2 = oracle.merge(pool[keep], inten[keep], origin[keep], rho)
    assert np.array_equal(keep2, np.arange(len(keep)))
    dup = oracle.merge(np.array([pool[0], pool[0]]), np.array([3, 3]), np.array([5, 9]), rho)
    assert dup.tolist() == [0]
    far = oracle.merge(np.eye(3), np.array([1, 2, 3]), np.array([0, 1, 2]), rho)
    assert far.tolist() == [2, 1, 0]


def test_assign_matches_numpy_and_sklearn():
    # P7: label = argmax_k x.c_k (ties lowest k) == nearest neighbour among unit centres
    rng = np.random.default_rng(9)
    X = _unit(rng.standard_normal((4000, 16)))
    Cn = _unit(rng.standard_normal((37, 16)))
    lab, cov, hist = oracle.assign(X, Cn, 0.1)
    assert np.array_equal(lab, np.argmax(X @ Cn.T, axis=1))
    nn = NearestNeighbors(n_neighbors=1).fit(Cn)
    assert np.array_equal(lab, nn.kneighbors(X, return_distance=False)[:, 0])
    assert np.array_equal(cov, ((X @ Cn.T).max(axis=1) >= 0.9).astype(np.uint8))
    assert np.array_equal(hist, np.bincount(lab, minlength=37))
    # exact tie -> lowest index
    lab2, _, _ = oracle.assign(np.array([[1.0, 0.0]]), np.array([[0.0, 1.0], [0.6, 0.8], [0.6, -0.8]]), 0.1)
    assert lab2.tolist() == [1]


# --------------------------------------------------------------------------------------------
# whole method: P4 closed-form centres, P5 exact recovery, OSOP behaviour, determinism
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(5))
def test_well_separated_closed_form_and_recovery(seed):
    f = synth.make_frame("C1", seed)
    X = oracle.normalize(f.emb)
    pol = oracle.policy(kind=oracle.SEEDS_FIXED, n_seeds=64, rng_seed=seed)
    r = oracle.cluster(f.emb, pol=pol)
    assert r.status == 0
    idx = oracle.select(np.ones(f.n, np.uint8), 64, seed, 0)
    seeded = set(f.truth[idx].tolist())
    closed = {k: _unit(X[f.truth == k].sum(0)) for k in range(f.cells + 1)}
    # P4: every centre is the closed-form mean direction of one true cluster
    for c in r.centres:
        assert max(float(c @ closed[k]) for k in closed) >= 1 - 1e-12
    if len(seeded) == f.cells + 1:
        # P5: every cluster received a seed -> exact recovery
        assert r.K == f.cells + 1 and _bijection(r.labels, f.truth)
        assert r.trace["round_iters"][0] == 2   # one update to the closed form, one to confirm


@pytest.mark.parametrize("seed", range(3))
def test_osop_recovers_well_separated_frames(seed):
    # P5 under OSOP: an unseeded cell's pixels are uncovered, hence re-seeded
    f = synth.make_frame("S1sep", seed)
    pol = oracle.policy(kind=oracle.SEEDS_OSOP, n_seeds=16, rng_seed=seed,
                        min_instance_px=min_instance_px(f.n), saturation_stop=0)
    r = oracle.cluster(f.emb, pol=pol)
    assert r.status == 0
    assert r.K == f.cells + 1 and _bijection(r.labels, f.truth)
    t = r.trace
    assert t["round_K"][0] == 16
    for r_ in range(1, t["rounds"]):                     # "N will be doubled"
        assert t["round_K"][r_] == min(sum(t["round_K"][:r_]), t["round_cand"][r_ - 1])
    assert t["round_cand"][-1] == 0 or t["seeds_total"] >= 2 * t["round_nmin"][-1]


def test_determinism_across_thread_counts(tmp_path):
    code = ("import numpy as np, oracle, synth, sys\n"
            "f = synth.make_frame('S1', 1)\n"
            "r = oracle.cluster(f.emb, pol=oracle.policy(min_instance_px=12, saturation_stop=1))\n"
            "np.save(sys.argv[1], np.concatenate([r.labels.astype(np.float64), r.centres.ravel()]))\n")
    outs = []
    for t in (1, 4):
        p = str(tmp_path / f"o{t}.npy")
        env = dict(os.environ, OMP_NUM_THREADS=str(t), PYTHONPATH=os.getcwd())
        subprocess.check_call([sys.executable, "-c", code, p], env=env)
        outs.append(np.load(p))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_session_carries_seed_count_between_frames():
    """NEXT-1 / O8: frame t+1's round 0 uses the seed count session_next() derived from frame t."""
    import synth
    from synth.frames import min_instance_px
    frames = [synth.make_frame("S1", s).emb for s in range(3)]
    pol = oracle.policy(min_instance_px=min_instance_px(frames[0].shape[0]), saturation_stop=1, n_seeds=32)
    res, Ns = oracle.session(frames, pol=pol)
    assert Ns[0] == 32 and all(r.status == 0 for r in res)
    for t in range(1, len(res)):
        prev = res[t - 1].trace
        assert Ns[t] == oracle.session_next(prev["seeds_total"], prev["round_nmin"][-1], pol.H)
        assert res[t].trace["round_K"][0] == min(Ns[t], frames[t].shape[0])
