"""Pixel sharding on one GPU: world_size-2/3 process groups over gloo share cuda:0.

Each rank holds a contiguous range of every frame's pixels (include/fms.h fms_set_pixel_shard); the
window sums G of every lockstep step, the seed rows, the mode intensities, the label histogram and the
coverage bits are summed through torch.distributed.  The method's result must not depend on the split:
the ranks' label slices, concatenated, and every rank's centres / K / per-round trace are bit-identical
to the unsharded run, and (well-separated frame) equal to the fp64 oracle.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import synth
from synth.frames import min_instance_px

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _policy_kw(cfg, n):
    if cfg == "C1":
        return dict(kind=0, n_seeds=64)
    if cfg == "ALL":
        return dict(kind=2)
    return dict(min_instance_px=min_instance_px(n), saturation_stop=1)


def _inputs(cfg, seeds):
    if cfg == "ALL":
        return np.stack([synth.make_blobs(1500, s)[0] for s in seeds])
    return np.stack([synth.make_frame(cfg, s).emb for s in seeds])


def _worker(rank, world, port, cfg, seeds, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_14283_b200 as fms
    from paper_2007_14283_b200.dist import enable_pixel_sharding
    X = _inputs(cfg, seeds)
    n = X.shape[1]
    ctx = fms.Context(0)
    lo, hi = enable_pixel_sharding(ctx, n)
    x = torch.from_numpy(np.ascontiguousarray(X[:, lo:hi])).cuda()
    pol = fms.default_policy(**_policy_kw(cfg, n))
    labels, centres, K, st = ctx.cluster(x, policy=pol, centres_cap=2048)
    np.savez(os.path.join(out, f"r{rank}.npz"), labels=labels.cpu().numpy(), centres=centres.cpu().numpy(),
             K=np.array(K), lo=lo, hi=hi, iters=np.array([f["seed_iters"] for f in st["frames"]]),
             rk=np.array([f["round_K"] for f in st["frames"]]), rc=np.array([f["round_conv"] for f in st["frames"]]),
             cand=np.array([f["round_cand"] for f in st["frames"]]))
    dist.barrier()
    dist.destroy_process_group()


def _run_sharded(cfg, seeds, world):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(world, _free_port(), cfg, seeds, out), nprocs=world, join=True,
                           start_method="spawn")
        return [dict(np.load(os.path.join(out, f"r{r}.npz"))) for r in range(world)]


def _run_single(cfg, seeds):
    import torch
    import paper_2007_14283_b200 as fms
    X = _inputs(cfg, seeds)
    x = torch.from_numpy(X).cuda()
    pol = fms.default_policy(**_policy_kw(cfg, X.shape[1]))
    labels, centres, K, st = fms.cluster(x, policy=pol, centres_cap=2048)
    return dict(labels=labels.cpu().numpy(), centres=centres.cpu().numpy(), K=np.array(K),
                iters=np.array([f["seed_iters"] for f in st["frames"]]),
                rk=np.array([f["round_K"] for f in st["frames"]]), rc=np.array([f["round_conv"] for f in st["frames"]]),
                cand=np.array([f["round_cand"] for f in st["frames"]]))


@pytest.mark.parametrize("cfg,seeds,world", [("S1", [0, 1], 2), ("S1", [2], 3), ("C2", [0], 2), ("C2sep", [0], 2),
                                             ("C1", [2], 2), ("S32sep", [0], 3), ("ALL", [0], 2)])
def test_pixel_sharded_equals_unsharded(cfg, seeds, world):
    ref = _run_single(cfg, seeds)
    parts = _run_sharded(cfg, seeds, world)
    assert [int(r["lo"]) for r in parts][0] == 0 and int(parts[-1]["hi"]) == ref["labels"].shape[1]
    labels = np.concatenate([r["labels"] for r in parts], axis=1)
    assert np.array_equal(labels, ref["labels"])
    for r in parts:
        for key in ("K", "iters", "rk", "rc", "cand", "centres"):
            assert np.array_equal(r[key], ref[key]), key


def test_pixel_sharded_matches_oracle_exact():
    import oracle
    from tests.parity_util import bijection, match_centres
    f = synth.make_frame("S1sep", 1)
    parts = _run_sharded("S1sep", [1], 2)
    labels = np.concatenate([r["labels"][0] for r in parts])
    pol = oracle.policy(kind=1, n_seeds=128, gamma=0.9, L=2.0, H=8.0, P=0.99, has_background=1,
                        min_instance_px=min_instance_px(f.n), saturation_stop=1, max_rounds=8, rng_seed=0)
    ro = oracle.cluster(f.emb, h=0.1, max_iter=300, tol=None, pol=pol)
    assert int(parts[0]["K"][0]) == ro.K
    assert bijection(labels, ro.labels)
    _, _, dist = match_centres(parts[1]["centres"][0, :ro.K], ro.centres)
    assert dist.max() <= 1e-4
