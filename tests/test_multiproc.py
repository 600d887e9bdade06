"""N>1 host logic on CPU with gloo (world_size 2): max-over-ranks timing reduction and the
rank-0-only reference arm of bench.py (frames are independent, so the GPU path is replicas)."""
import json
import os
import re
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
sys.stdout.write(f"RESULT {r} {v}\n"); sys.stdout.flush()
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
    # the two ranks share stdout, so lines may interleave: match the records anywhere
    res = re.findall(r"RESULT (\d+) ([0-9.]+)", out.stdout)
    assert sorted(int(r) for r, _ in res) == [0, 1] and all(float(v) == 15.0 for _, v in res), out.stdout


def test_reference_arm_rank0_only():
    out = _torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                     "--config", "S1"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
