"""CUDA path (libfms.so through its C ABI) vs the fp64 oracle on identical seeded inputs.

Bar (BASELINE.json north_star): well-separated frames -> equal K, labels identical up to a cluster
permutation, centres within 1e-4 cosine distance, identical per-round trace; near-boundary frames ->
ARI >= 0.999 and centres of clusters >= min_instance_px within 1e-4.
"""
import numpy as np
import pytest

import oracle
import synth
from synth.frames import min_instance_px
from tests.parity_util import ari, bijection, match_centres

pytestmark = pytest.mark.gpu


def _fms():
    import paper_2007_14283_b200 as fms
    return fms


def run_gpu(emb, h=0.1, cap=4096, max_iters=300, tol=None, allow=(), **pol):
    import torch
    fms = _fms()
    x = torch.from_numpy(np.ascontiguousarray(emb, dtype=np.float32)).cuda()
    labels, centres, K, st = fms.cluster(x, h=h, max_iters=max_iters, tol=tol, policy=fms.default_policy(**pol),
                                         centres_cap=cap, allow=allow)
    torch.cuda.synchronize()
    return labels.cpu().numpy(), centres.cpu().numpy(), K, st


def run_orc(emb, h=0.1, max_iters=300, tol=None, **pol):
    base = dict(kind=1, n_seeds=128, gamma=0.9, L=2.0, H=8.0, P=0.99, has_background=1, min_instance_px=0,
                saturation_stop=0, max_rounds=8, rng_seed=0)
    base.update(pol)
    return oracle.cluster(emb, h=h, max_iter=max_iters, tol=tol, pol=oracle.policy(**base))


def check_exact(emb, h=0.1, trace=True, **pol):
    lg, cg, Kg, st = run_gpu(emb, h=h, **pol)
    ro = run_orc(emb, h=h, **pol)
    assert ro.status == 0
    assert Kg[0] == ro.K, (Kg, ro.K, st["frames"][0], ro.trace)
    assert bijection(lg[0], ro.labels)
    r, c, dist = match_centres(cg[0, :Kg[0]], ro.centres)
    assert dist.max() <= 1e-4, dist.max()
    if trace:
        fg = st["frames"][0]
        for key in ("rounds", "round_K", "round_iters", "round_conv", "round_Kc"):
            assert fg[key] == ro.trace[key], (key, fg[key], ro.trace[key])
    return lg, cg, Kg, st, ro


def check_near(emb, h=0.1, min_ari=0.999, **pol):
    lg, cg, Kg, st = run_gpu(emb, h=h, **pol)
    ro = run_orc(emb, h=h, **pol)
    assert ro.status == 0
    a = ari(lg[0], ro.labels)
    assert a >= min_ari, (a, Kg, ro.K, st["frames"][0], ro.trace)
    big = np.nonzero(np.bincount(ro.labels, minlength=ro.K) >= max(1, pol.get("min_instance_px", 1)))[0]
    r, c, dist = match_centres(cg[0, :Kg[0]], ro.centres[big])
    assert dist.max() <= 1e-4, dist.max()
    return a


# ---------------------------------------------------------------------------------------------
# well-separated frames: exact
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(5))
def test_c1_fixed64_exact(seed):
    f = synth.make_frame("C1", seed)
    check_exact(f.emb, kind=0, n_seeds=64, rng_seed=seed)


def test_single_lockstep_step_exact():
    # one K2+K3 step: tol so large that every seed converges after its first update
    f = synth.make_frame("C1", 7)
    lg, cg, Kg, st = run_gpu(f.emb, tol=10.0, kind=0, n_seeds=64, gamma=1.0)
    ro = run_orc(f.emb, tol=10.0, kind=0, n_seeds=64, gamma=1.0)
    assert st["frames"][0]["round_iters"] == [1] == ro.trace["round_iters"]
    assert Kg[0] == ro.K and bijection(lg[0], ro.labels)
    assert match_centres(cg[0, :Kg[0]], ro.centres)[2].max() <= 1e-4


@pytest.mark.parametrize("seed", range(3))
def test_s1sep_osop_exact(seed):
    f = synth.make_frame("S1sep", seed)
    check_exact(f.emb, n_seeds=16, rng_seed=seed, min_instance_px=min_instance_px(f.n))


def test_s32sep_d32_exact():
    f = synth.make_frame("S32sep", 0)
    check_exact(f.emb, n_seeds=32, rng_seed=1, min_instance_px=min_instance_px(f.n))


def test_c2sep_full_size_exact():
    f = synth.make_frame("C2sep", 0)
    check_exact(f.emb, rng_seed=0, min_instance_px=min_instance_px(f.n), saturation_stop=1)


# ---------------------------------------------------------------------------------------------
# near-boundary frames: ARI
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(3))
def test_s1_soft_osop_ari(seed):
    f = synth.make_frame("S1", seed)
    check_near(f.emb, rng_seed=seed, min_instance_px=min_instance_px(f.n), saturation_stop=1)


@pytest.mark.parametrize("seed", range(2))
def test_c2_full_size_ari(seed):
    f = synth.make_frame("C2", seed)
    check_near(f.emb, rng_seed=seed, min_instance_px=min_instance_px(f.n), saturation_stop=1)


def test_c3_nonsquare_ari():
    f = synth.make_frame("C3_simplus", 0)
    check_near(f.emb, rng_seed=0, min_instance_px=min_instance_px(f.n), saturation_stop=1)


def _many_clusters(k=200, per=80, d=16, seed=7):
    """k well-separated directions (pairwise cosine < 0.7), `per` pixels each within cosine 0.97."""
    rng = np.random.default_rng(seed)
    dirs = []
    while len(dirs) < k:
        v = rng.standard_normal(d)
        v /= np.linalg.norm(v)
        if all(abs(float(v @ u)) < 0.7 for u in dirs):
            dirs.append(v)
    dirs = np.array(dirs)
    pts = []
    for c in range(k):
        noise = rng.standard_normal((per, d)) * 0.04
        x = dirs[c] + noise
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        pts.append(x)
    emb = np.concatenate(pts)[rng.permutation(k * per)]
    return emb.astype(np.float32)


def test_more_than_128_modes_exact():
    """> 128 modes: the last rounds' assignment runs on the CUDA-core kernel, earlier ones on the
    tensor cores -- both must reproduce the oracle exactly (Alg. 2 l.12-14)."""
    emb = _many_clusters()
    lg, cg, Kg, st, ro = check_exact(emb, rng_seed=3, has_background=0)
    assert ro.K > 128 and max(ro.trace["round_Kc"]) > 128


def test_c5_small_stack_ari():
    """C5-shaped joint clustering of a temporal stack (tracks drift and their directions random-walk)
    at a size the oracle finishes: 6 frames of 128x128, 8 tracks."""
    emb, _ = synth.make_stack(6, seed=2, H=128, W=128, cells=8, radius=(10, 18))
    check_near(emb, rng_seed=0, min_instance_px=6 * min_instance_px(128 * 128), saturation_stop=1)


@pytest.mark.parametrize("n,kind", [(1000, 2), (2000, 2), (5000, 1), (9000, 2)])
def test_table1_blobs_exact(n, kind):
    """NEXT-3: the paper's Table 1 simulation data (18-D blobs, 10 orthogonal/opposite
    clusters, noise 0.01) under Alg. 1 (kind 2, every point a seed) and OSOP: exact vs the oracle."""
    emb, _ = synth.make_blobs(n, seed=1)
    check_exact(emb, kind=kind, n_seeds=128, has_background=0)


# ---------------------------------------------------------------------------------------------
# batching, determinism, host entry
# ---------------------------------------------------------------------------------------------

def test_batch_equals_single_and_deterministic():
    import torch
    fms = _fms()
    frames = [synth.make_frame("S1", s) for s in range(3)]
    X = torch.from_numpy(np.stack([f.emb for f in frames])).cuda()
    pol = fms.default_policy(min_instance_px=min_instance_px(frames[0].n), saturation_stop=1)
    lb, cb, Kb, _ = fms.cluster(X, policy=pol, centres_cap=512)
    lb2, cb2, Kb2, _ = fms.cluster(X, policy=pol, centres_cap=512)
    assert Kb == Kb2 and torch.equal(lb, lb2) and torch.equal(cb, cb2)
    for b, f in enumerate(frames):
        l1, c1, K1, _ = fms.cluster(X[b], policy=pol, centres_cap=512)
        assert K1[0] == Kb[b]
        assert torch.equal(l1[0], lb[b]) and torch.equal(c1[0], cb[b])


def test_host_entry_matches_device_entry():
    import torch
    fms = _fms()
    f = synth.make_frame("S1", 5)
    pol = fms.default_policy(min_instance_px=min_instance_px(f.n), saturation_stop=1)
    ld, cd, Kd, _ = fms.cluster(torch.from_numpy(f.emb).cuda(), policy=pol, centres_cap=256)
    eh = torch.from_numpy(f.emb).reshape(1, f.n, f.D).pin_memory()
    lh = torch.empty((1, f.n), dtype=torch.int32).pin_memory()
    ch = torch.zeros((1, 256, f.D), dtype=torch.float32).pin_memory()
    rc, Kh, rs = fms.context(0).cluster_host(eh, lh, ch, 256, policy=pol)
    assert Kh == Kd
    assert torch.equal(lh, ld.cpu()) and torch.equal(ch, cd.cpu())


def test_host_entry_chunked_overlap_matches_device_entry():
    # 5 frames in chunks of 2 (ragged last chunk): uploads, compute and downloads overlap on two streams
    import torch
    fms = _fms()
    frames = [synth.make_frame("S1", 10 + s) for s in range(5)]
    X = np.stack([f.emb for f in frames])
    pol = fms.default_policy(min_instance_px=min_instance_px(frames[0].n), saturation_stop=1)
    ld, cd, Kd, _ = fms.cluster(torch.from_numpy(X).cuda(), policy=pol, centres_cap=128)
    ctx = fms.Context(0)
    ctx.set_option("host_chunk", 2)
    eh = torch.from_numpy(X).pin_memory()
    lh = torch.full((5, frames[0].n), -1, dtype=torch.int32).pin_memory()
    ch = torch.zeros((5, 128, frames[0].D), dtype=torch.float32).pin_memory()
    for _ in range(2):  # the second call reuses the staging buffers
        rc, Kh, rs = ctx.cluster_host(eh, lh, ch, 128, policy=pol)
        assert Kh == Kd
        assert torch.equal(lh, ld.cpu()) and torch.equal(ch, cd.cpu())


# ---------------------------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------------------------

def _blobs(n_per, k, d, noise, seed, bg=0):
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((k, d))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    X = np.concatenate([C[j] + noise * rng.standard_normal((n_per, d)) for j in range(k)]
                       + [rng.standard_normal((bg, d))])
    return (X * rng.uniform(0.5, 2, (X.shape[0], 1))).astype(np.float32)


@pytest.mark.parametrize("d", [3, 5, 18, 32])
def test_ragged_n_and_padded_d(d):
    X = _blobs(311, 3, d, 0.01, d)          # n = 933: not a multiple of the 128-pixel tile
    check_exact(X, kind=0, n_seeds=40, rng_seed=3)


def test_tiny_inputs():
    lg, cg, Kg, st = run_gpu(np.array([[3.0, 4.0]], dtype=np.float32), kind=0, n_seeds=8)
    assert Kg[0] == 1 and lg[0].tolist() == [0]
    assert 1.0 - cg[0, 0] @ np.array([0.6, 0.8]) <= 1e-4   # cosine-distance parity bar
    X = _blobs(2, 2, 4, 0.0, 1)
    check_exact(X, kind=0, n_seeds=64)


def test_all_points_mode_alg1():
    X = _blobs(100, 3, 6, 0.03, 11, bg=0)
    check_exact(X, kind=2, trace=False)


def test_errors():
    fms = _fms()
    X = _blobs(50, 2, 4, 0.01, 2)
    X[7] = 0.0
    with pytest.raises(fms.FmsError) as e:
        run_gpu(X, kind=0, n_seeds=8)
    assert e.value.status == 3
    with pytest.raises(fms.FmsError) as e:
        run_gpu(_blobs(50, 2, 4, 0.01, 2), h=1.5)
    assert e.value.status == 2
    with pytest.raises(fms.FmsError) as e:
        run_gpu(_blobs(50, 2, 40, 0.01, 2))
    assert e.value.status == 2


def test_capacity_reports_required_k():
    fms = _fms()
    f = synth.make_frame("C1", 0)
    lg, cg, Kg, st = run_gpu(f.emb, cap=2, allow=(5,), kind=0, n_seeds=64)
    assert st["status"] == 5 and Kg[0] == 6
