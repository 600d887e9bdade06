"""N>1 host logic on CPU with gloo (world_size 2): max-over-ranks timing reduction and the
rank-0-only reference arm of bench.py (frames are independent, so the GPU path is replicas)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r"""
import os, sys
sys.path.insert(0, %r)
import torch.distributed as dist
dist.init_process_group("gloo")
import bench
r = dist.get_rank()
v = bench.reduce_max(10.0 + 5.0 * r, dist.get_world_size())
print("RESULT", r, v, flush=True)
dist.destroy_process_group()
"""


def _torchrun(args, timeout=300):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=ROOT, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000)] + args
    return subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


def test_reduce_max_over_two_ranks(tmp_path):
    w = tmp_path / "w.py"
    w.write_text(_WORKER % ROOT)
    out = _torchrun([str(w)])
    assert out.returncode == 0, out.stderr[-2000:]
    res = [l.split() for l in out.stdout.splitlines() if l.startswith("RESULT")]
    assert len(res) == 2 and all(float(x[2]) == 15.0 for x in res)


def test_reference_arm_rank0_only():
    out = _torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                     "--config", "S1"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
