"""Feature combinations on the CUDA path: the NEXT-4 variants through the other entry points
(host-buffer entry with overlapped copies, frame sessions, seed sharding)."""
import os
import socket
import tempfile

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


def test_euclid_host_entry_matches_device_entry():
    import torch
    import paper_2007_14283_b200 as fms
    X = np.stack([_blobs(5, 200, 8, 0.1, 3.0, seed=s, scale=7.0) for s in range(3)])
    ctx = fms.Context(0)
    ctx.set_option("metric", 1)
    ctx.set_option("host_chunk", 2)
    pol = fms.default_policy(kind=0, n_seeds=32, gamma=1.0, has_background=0)
    ld, cd, Kd, _ = ctx.cluster(torch.from_numpy(X).cuda(), h=4.0, policy=pol, centres_cap=64)
    eh = torch.from_numpy(X).pin_memory()
    lh = torch.empty((3, X.shape[1]), dtype=torch.int32).pin_memory()
    ch = torch.zeros((3, 64, 8), dtype=torch.float32).pin_memory()
    rc, Kh, _ = ctx.cluster_host(eh, lh, ch, 64, h=4.0, policy=pol)
    assert Kh == Kd and torch.equal(lh, ld.cpu()) and torch.equal(ch, cd.cpu())
    # centres come back in the caller's units (the data were scaled by 7)
    for b in range(3):
        ro = oracle.cluster(X[b], h=4.0, pol=oracle.policy(kind=0, n_seeds=32, gamma=1.0, has_background=0,
                                                            metric=oracle.METRIC_EUCLID))
        D = np.linalg.norm(cd.cpu().numpy()[b, :Kd[b], None, :] - ro.centres[None, :, :], axis=2)
        assert D.min(axis=1).max() <= 1e-4 * 4.0


def test_euclid_session_matches_oracle_session():
    import torch
    import paper_2007_14283_b200 as fms
    frames = [_blobs(6, 300, 10, 0.1, 3.0, seed=20 + t) for t in range(3)]
    opol = oracle.policy(n_seeds=16, has_background=0, metric=oracle.METRIC_EUCLID)
    ro, Ns = oracle.session(frames, h=0.9, pol=opol)
    ctx = fms.Context(0)
    ctx.set_option("metric", 1)
    sess = fms.Session(ctx, fms.default_policy(n_seeds=16, has_background=0))
    for t, emb in enumerate(frames):
        assert sess.seeds == Ns[t]
        labels, centres, K, fs = sess.step(torch.from_numpy(emb).cuda(), h=0.9, centres_cap=256)
        assert K == ro[t].K and fs["round_K"] == ro[t].trace["round_K"]
        assert bijection(labels.cpu().numpy(), ro[t].labels)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_14283_b200 as fms
    import synth
    from paper_2007_14283_b200.dist import enable_seed_sharding
    from synth.frames import min_instance_px
    f = synth.make_frame("S1", 3)
    ctx = enable_seed_sharding(fms.Context(0))
    ctx.set_option("kernel_profile", 1)
    pol = fms.default_policy(min_instance_px=min_instance_px(f.n), saturation_stop=1)
    labels, centres, K, st = ctx.cluster(torch.from_numpy(f.emb).cuda(), policy=pol, centres_cap=256)
    np.savez(os.path.join(out, f"r{rank}.npz"), labels=labels.cpu().numpy(), centres=centres.cpu().numpy(),
             K=np.array(K))
    dist.barrier()
    dist.destroy_process_group()


def test_gauss_seed_sharded_equals_unsharded():
    import torch
    import torch.multiprocessing as mp
    import paper_2007_14283_b200 as fms
    import synth
    from synth.frames import min_instance_px
    f = synth.make_frame("S1", 3)
    ctx = fms.Context(0)
    ctx.set_option("kernel_profile", 1)
    pol = fms.default_policy(min_instance_px=min_instance_px(f.n), saturation_stop=1)
    l1, c1, K1, _ = ctx.cluster(torch.from_numpy(f.emb).cuda(), policy=pol, centres_cap=256)
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
        for r in range(2):
            d = dict(np.load(os.path.join(out, f"r{r}.npz")))
            assert np.array_equal(d["K"], np.array(K1))
            assert np.array_equal(d["labels"], l1.cpu().numpy())
            assert np.array_equal(d["centres"], c1.cpu().numpy())
