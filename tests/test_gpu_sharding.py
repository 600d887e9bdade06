"""Seed sharding on one GPU: world_size-2 process groups over gloo share cuda:0.

Each rank iterates only its share of every round's seeds (include/fms.h fms_set_exchange); the
per-step counts and the per-round converged seeds are summed through torch.distributed.  The
method's result must not depend on the split: every rank returns labels / centres / K / per-round
trace bit-identical to the unsharded run, and (well-separated frame) equal to the fp64 oracle.
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
    return dict(min_instance_px=min_instance_px(n), saturation_stop=1)


def _worker(rank, world, port, cfg, seeds, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_14283_b200 as fms
    from paper_2007_14283_b200.dist import enable_seed_sharding
    frames = [synth.make_frame(cfg, s) for s in seeds]
    ctx = enable_seed_sharding(fms.Context(0))
    x = torch.from_numpy(np.stack([f.emb for f in frames])).cuda()
    pol = fms.default_policy(**_policy_kw(cfg, frames[0].n))
    labels, centres, K, st = ctx.cluster(x, policy=pol, centres_cap=1024)
    np.savez(os.path.join(out, f"r{rank}.npz"), labels=labels.cpu().numpy(), centres=centres.cpu().numpy(),
             K=np.array(K), iters=np.array([f["seed_iters"] for f in st["frames"]]),
             rk=np.array([f["round_K"] for f in st["frames"]]), rc=np.array([f["round_conv"] for f in st["frames"]]))
    dist.barrier()
    dist.destroy_process_group()


def _run_sharded(cfg, seeds, world=2):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(world, _free_port(), cfg, seeds, out), nprocs=world, join=True,
                           start_method="spawn")
        return [dict(np.load(os.path.join(out, f"r{r}.npz"))) for r in range(world)]


def _run_single(cfg, seeds):
    import torch
    import paper_2007_14283_b200 as fms
    frames = [synth.make_frame(cfg, s) for s in seeds]
    x = torch.from_numpy(np.stack([f.emb for f in frames])).cuda()
    pol = fms.default_policy(**_policy_kw(cfg, frames[0].n))
    labels, centres, K, st = fms.cluster(x, policy=pol, centres_cap=1024)
    return dict(labels=labels.cpu().numpy(), centres=centres.cpu().numpy(), K=np.array(K),
                iters=np.array([f["seed_iters"] for f in st["frames"]]),
                rk=np.array([f["round_K"] for f in st["frames"]]), rc=np.array([f["round_conv"] for f in st["frames"]]))


@pytest.mark.parametrize("cfg,seeds", [("S1", [0, 1]), ("C2sep", [0]), ("C1", [2])])
def test_seed_sharded_equals_unsharded(cfg, seeds):
    ref = _run_single(cfg, seeds)
    for r in _run_sharded(cfg, seeds):
        for key in ("K", "iters", "rk", "rc", "labels", "centres"):
            assert np.array_equal(r[key], ref[key]), key


def test_seed_sharded_matches_oracle_exact():
    import oracle
    from tests.parity_util import bijection, match_centres
    f = synth.make_frame("S1sep", 1)
    r = _run_sharded("S1sep", [1])[0]
    pol = oracle.policy(kind=1, n_seeds=128, gamma=0.9, L=2.0, H=8.0, P=0.99, has_background=1,
                        min_instance_px=min_instance_px(f.n), saturation_stop=1, max_rounds=8, rng_seed=0)
    ro = oracle.cluster(f.emb, h=0.1, max_iter=300, tol=None, pol=pol)
    assert int(r["K"][0]) == ro.K
    assert bijection(r["labels"][0], ro.labels)
    _, _, dist = match_centres(r["centres"][0, :ro.K], ro.centres)
    assert dist.max() <= 1e-4


def _nccl_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_14283_b200 as fms
    from paper_2007_14283_b200.dist import enable_seed_sharding
    f = synth.make_frame("S1sep", 1)
    ctx = fms.Context(0)
    result = {}
    try:
        enable_seed_sharding(ctx, in_library=True)   # fms_nccl_unique_id + fms_set_nccl over 2 ranks
        labels, centres, K, st = ctx.cluster(torch.from_numpy(f.emb).cuda(),
                                             policy=fms.default_policy(**_policy_kw("S1sep", f.n)),
                                             centres_cap=1024)
        result = dict(ok=1, labels=labels.cpu().numpy(), K=np.array(K))
    except fms.FmsError as e:
        result = dict(ok=0, status=e.status, msg=str(e))
    np.save(os.path.join(out, f"n{rank}.npy"), result, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_in_library_nccl_two_ranks():
    """In-library NCCL (include/fms.h fms_set_nccl): rank 0's unique id is shared through
    torch.distributed and both ranks build the communicator.  With two ranks on ONE GPU, NCCL either
    runs (then the result equals the unsharded run) or refuses the duplicate device -- the library
    must report that as FMS_E_NCCL with NCCL's message, not hang or crash."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_nccl_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
        res = [np.load(os.path.join(out, f"n{r}.npy"), allow_pickle=True).item() for r in range(2)]
    print("in-library NCCL, 2 ranks on one GPU:", [("ran" if r["ok"] else r.get("msg")) for r in res])
    if all(r["ok"] for r in res):
        ref = _run_single("S1sep", [1])
        for r in res:
            assert np.array_equal(r["labels"], ref["labels"]) and np.array_equal(r["K"], ref["K"])
    else:
        for r in res:
            assert r["ok"] or (r["status"] == 7 and "nccl" in r["msg"].lower()), r
