"""Benchmark of the Faster Mean-shift hot path on B200 (one JSON line on rank 0).

metric: frames/sec clustering 512x512 frames of 16-D embeddings (BASELINE.json configs[1], the
        metric config: ~30 touching/overlapping cells, full OSOP), plus the iteration kernel's
        fraction of its tensor roofline.
step  : one call of fms_cluster_batch on a batch of B resident frames (every §8(a) row runs:
        normalise, select, lockstep iteration, intensity, merge, assign, OSOP control).
multi-GPU: frames are independent (replicas, no data-path collective); each rank
        clusters its own batches; the elapsed time is the max over ranks.  N > 1 runs add two strong-
        scaling measurements: C4 seed-sharded (8(e) 2) and the C5 stack pixel-sharded (8(e) 3).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl fms|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "C2"
H = 0.1
MAX_ITERS = 300
CAP = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=96)  # frames in flight: 32 -> 1319, 64 -> 1399, 96 -> 1441, 128 -> 1415 frames/s
    ap.add_argument("--impl", default="fms", choices=["fms", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0,
                    help="cpu_baseline: seconds of oracle work per thread setting (nproc, then 1 thread)")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "seeds"],
                    help="replicas: every rank clusters its own frames (weak scaling); seeds: every rank "
                         "clusters the same frames and iterates 1/N of each round's seeds (strong scaling, "
                         "SURVEY 8(e)2; exchange through torch.distributed)")
    ap.add_argument("--kernel-profile", default="flat", choices=["flat", "gauss"],
                    help="kernel of the mean-shift update: the paper's flat kernel, or the Gaussian profile "
                         "(NEXT-4, reading R23; SFU-bound)")
    ap.add_argument("--metric", default="cosine", choices=["cosine", "euclid"],
                    help="euclid (NEXT-4, reading R24): the C2 frames row-normalised, Euclidean window "
                         "sqrt(2h) (the same windows as cosine h at the start), window-mean update")
    ap.add_argument("--host-chunk", type=int, default=0, help="e2e: frames per host-entry chunk (0 = library default)")
    ap.add_argument("--no-pdl", action="store_true", help="launch the step kernels without programmatic dependent launch")
    ap.add_argument("--fuse-step", type=int, default=0, choices=[0, 1],
                    help="graph step tail as one kernel (1; measured slower) or update / ctl / cond / plan kernels (0, default)")
    ap.add_argument("--extras-budget-s", type=float, default=300.0,
                    help="N > 1: time budget of the sharded extra measurements")
    ap.add_argument("--no-seed-shard", action="store_true",
                    help="with N > 1 replicas: skip the extra seed-sharded C4 measurement")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend of the fms arm (gloo: several ranks may share one GPU)")
    return ap.parse_args()


def policy_kwargs(n):
    from synth.frames import min_instance_px
    return dict(min_instance_px=min_instance_px(n), saturation_stop=1)


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "fms":
            torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group(args.backend)
        else:
            dist.init_process_group("gloo")
    return world, rank, local


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 50 ms) during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.err = None

    def _run(self):
        import pynvml
        try:
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self.stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append((sm, mx, rs, util))
                self.stop.wait(0.05)
        except Exception as e:  # pragma: no cover
            self.err = repr(e)

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=5)

    def summary(self):
        rows = [r for r in self.rows if r[3] > 0] or self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        sm = sorted(r[0] for r in rows)
        reasons = sorted({name for r in rows for bit, name in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def reduce_max(x: float, world: int, device=None) -> float:
    """Max over ranks of a per-rank time (barrier first); identity on one rank."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.barrier()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return m, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic():
    """dram bytes per K2 launch from the committed ncu --set full summary, if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "k2_ncu.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


_CPU_CODE = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
import oracle, synth
from synth.frames import min_instance_px
cfg, first, budget, h, max_iter = sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), float(sys.argv[5]), int(sys.argv[6])
done, sit, t0, i = 0, 0, time.perf_counter(), first
while True:
    f = synth.make_frame(cfg, i)
    r = oracle.cluster(f.emb, h=h, max_iter=max_iter,
                       pol=oracle.policy(rng_seed=0, min_instance_px=min_instance_px(f.n), saturation_stop=1))
    assert r.status == 0
    done += 1
    sit += r.trace["seed_iters"]
    i += 1
    if time.perf_counter() - t0 > budget:
        break
print(json.dumps({"frames": done, "seconds": time.perf_counter() - t0, "seed_iters": sit,
                  "threads": oracle.lib().fmso_num_threads(), "seeds": [first, i - 1]}))
"""


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_run(config, first, budget_s, threads):
    """The oracle as it stands (plain C, fp64, OpenMP over seeds/pixels) in a child process with
    OMP_NUM_THREADS=threads on frames first, first+1, ... of the GPU arm's own pool (the same
    generator seeds) until budget_s is spent (at least one frame)."""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    p = subprocess.run([sys.executable, "-c", _CPU_CODE, ROOT, config, str(first), str(budget_s), str(H),
                        str(MAX_ITERS)], capture_output=True, text=True, env=env, timeout=budget_s * 20 + 600)
    return json.loads(p.stdout.strip().splitlines()[-1])


def cpu_baseline(config, budget_s=20.0, first=0):
    """cpu_baseline of the JSON line (rank 0, N = 1): the oracle on the host cores at nproc threads
    and at 1 thread, each on a bounded sample of the GPU arm's own frames (pool seeds 0, 1, ...).
    Per-frame work varies several-fold between frames, so the seed-iterations per second (the
    algorithmic work rate) are reported beside frames/s."""
    nproc = os.cpu_count() or 1
    full = cpu_run(config, first, budget_s, nproc)
    one = cpu_run(config, first, budget_s, 1)
    return {"value": full["frames"] / full["seconds"], "unit": "frames/s", "cores": full["threads"],
            "kind": "oracle",
            "sample": f"{config} frames of the GPU pool, generator seeds {full['seeds'][0]}..{full['seeds'][1]} "
                      f"({full['frames']} frame(s), {full['seconds']:.1f} s), fp64 C oracle, OpenMP",
            "seed_iters_per_s": full["seed_iters"] / full["seconds"],
            "one_thread": {"value": one["frames"] / one["seconds"], "unit": "frames/s", "cores": 1,
                           "seed_iters_per_s": one["seed_iters"] / one["seconds"],
                           "sample": f"generator seeds {one['seeds'][0]}..{one['seeds'][1]} ({one['frames']} "
                                     f"frame(s), {one['seconds']:.1f} s)"},
            "cpu_model": cpu_model(), "nproc": nproc}


def latency_and_b16(ctx, pool, pol, h_run, stream, reps=20):
    """SURVEY 8(d) timing protocol extras (one GPU): single-frame latency (median / p90 over `reps`
    calls, each frame a different pool frame) with the input resident and through the host-buffer
    entry (H2D + D2H inside the call), and batched throughput at B = 16, both ways."""
    import numpy as np
    import torch
    dev = pool.device
    B2, n, d = pool.shape[1], pool.shape[2], pool.shape[3]
    flat = pool.reshape(-1, n, d)
    lab = torch.empty((16, n), dtype=torch.int32, device=dev)
    cen = torch.empty((16, CAP, d), dtype=torch.float32, device=dev)
    out = {}

    def dev_call(x, Bx):
        ctx.cluster_batch_ptr(x.data_ptr(), Bx, n, d, lab.data_ptr(), cen.data_ptr(), CAP, h_run, MAX_ITERS, None,
                              pol, stream.cuda_stream)

    lat = []
    for r in range(reps + 2):
        x = flat[r % flat.shape[0]]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dev_call(x, 1)
        e1.record(stream)
        torch.cuda.synchronize()
        if r >= 2:
            lat.append(e0.elapsed_time(e1))
    eh = flat[:16].cpu().pin_memory()
    lh = torch.empty((16, n), dtype=torch.int32).pin_memory()
    ch = torch.empty((16, CAP, d), dtype=torch.float32).pin_memory()
    lat_h = []
    for r in range(reps + 2):
        t0 = time.perf_counter()
        ctx.cluster_host(eh[r % 16:r % 16 + 1], lh[:1], ch[:1], CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
        torch.cuda.synchronize()
        if r >= 2:
            lat_h.append((time.perf_counter() - t0) * 1e3)
    q = lambda v, p: float(np.percentile(np.array(v), p))  # noqa: E731
    out["latency_ms"] = {"median": q(lat, 50), "p90": q(lat, 90), "calls": reps,
                         "entry": "fms_cluster_batch, B = 1, input resident (CUDA events)"}
    out["latency_e2e_ms"] = {"median": q(lat_h, 50), "p90": q(lat_h, 90), "calls": reps,
                             "entry": "fms_cluster_batch_host, B = 1, pinned host buffers (host wall clock)"}
    # B = 16 throughput: 5 steps over two alternating 16-frame batches
    x16 = [flat[:16], flat[16:32] if flat.shape[0] >= 32 else flat[:16]]
    dev_call(x16[0], 16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(5):
        dev_call(x16[k % 2], 16)
    e1.record(stream)
    torch.cuda.synchronize()
    out["b16"] = {"value": 80 / (e0.elapsed_time(e1) / 1e3), "unit": "frames/s", "steps": 5, "frames_per_step": 16}
    ctx.cluster_host(eh, lh, ch, CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(5):
        ctx.cluster_host(eh, lh, ch, CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    out["b16_e2e"] = {"value": 80 / (e0.elapsed_time(e1) / 1e3), "unit": "frames/s", "steps": 5,
                      "h2d_bytes_per_step": 16 * n * d * 4, "d2h_bytes_per_step": 16 * n * 4 + 16 * CAP * d * 4}
    return out


def seed_sharded_c4(world, rank, local, B=2, warmup=1, steps=3):
    """SURVEY 8(e)2 / BASELINE configs[3]: the same C4 frames (1024x1024, 32-D, ~200 cells) on every
    rank, each rank iterating 1/world of every round's seeds (strong scaling), next to the same
    frames clustered by one rank alone.  Device time, max over ranks."""
    import numpy as np
    import torch

    import paper_2007_14283_b200 as fms
    import synth
    from paper_2007_14283_b200.dist import enable_seed_sharding
    dev = torch.device("cuda", local)
    frames = [synth.make_frame("C4", 30000 + i) for i in range(B)]
    n, d = frames[0].n, frames[0].D
    x = torch.from_numpy(np.stack([f.emb for f in frames])).to(dev)
    labels = torch.empty((B, n), dtype=torch.int32, device=dev)
    cent = torch.empty((B, CAP, d), dtype=torch.float32, device=dev)
    pol = fms.default_policy(**policy_kwargs(n))
    stream = torch.cuda.current_stream(dev)

    def timed(ctx):
        Ks = None
        for _ in range(warmup):
            ctx.cluster_batch_ptr(x.data_ptr(), B, n, d, labels.data_ptr(), cent.data_ptr(), CAP, H, MAX_ITERS, None,
                                  pol, stream.cuda_stream)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            _, Ks, _, _ = ctx.cluster_batch_ptr(x.data_ptr(), B, n, d, labels.data_ptr(), cent.data_ptr(), CAP, H,
                                                MAX_ITERS, None, pol, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return reduce_max(e0.elapsed_time(e1), world, dev), Ks

    single_ms, K1 = timed(fms.Context(local))
    if world == 1:  # the one-GPU point of the C4 strong-scaling curve (N > 1 runs add the sharded points)
        return {"config": "C4: 1024x1024, 32-D, 200 cells, full OSOP", "frames_per_step": B, "n_gpus": 1,
                "value": steps * B / (single_ms / 1e3), "unit": "frames/s", "scaling": "strong"}
    sharded_ms, KN = timed(enable_seed_sharding(fms.Context(local)))
    return {"config": "C4: 1024x1024, 32-D, 200 cells, full OSOP", "frames_per_step": B, "n_gpus": world,
            "value": steps * B / (sharded_ms / 1e3), "unit": "frames/s", "scaling": "strong",
            "one_rank_value": steps * B / (single_ms / 1e3), "K_equal_to_one_rank": K1 == KN}


def pixel_sharded_c5(world, rank, local, T=92, warmup=1, steps=3):
    """SURVEY 8(e)3 / BASELINE configs[4]: the C5 temporal stack (T x 512x512, 16-D, ~30 tracks)
    clustered jointly as one problem, its pixels split over the ranks (fms_set_pixel_shard: per
    lockstep step an all-reduce of the exact window sums), next to the whole stack clustered by one
    rank alone (strong scaling).  Device time, max over ranks; checks that K and this rank's labels
    equal the one-rank run."""
    import numpy as np
    import torch

    import paper_2007_14283_b200 as fms
    import synth
    from paper_2007_14283_b200.dist import enable_pixel_sharding
    from synth.frames import min_instance_px
    dev = torch.device("cuda", local)
    emb, _ = synth.make_stack(T, seed=0)
    n, d = emb.shape
    pol = fms.default_policy(min_instance_px=min_instance_px(512 * 512) * T, saturation_stop=1)
    stream = torch.cuda.current_stream(dev)

    def timed(ctx, x):
        nl = x.shape[0]
        labels = torch.empty((1, nl), dtype=torch.int32, device=dev)
        cent = torch.empty((1, CAP, d), dtype=torch.float32, device=dev)
        Ks = None
        for _ in range(warmup):
            ctx.cluster_batch_ptr(x.data_ptr(), 1, nl, d, labels.data_ptr(), cent.data_ptr(), CAP, H, MAX_ITERS,
                                  None, pol, stream.cuda_stream)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            _, Ks, _, _ = ctx.cluster_batch_ptr(x.data_ptr(), 1, nl, d, labels.data_ptr(), cent.data_ptr(), CAP, H,
                                                MAX_ITERS, None, pol, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return reduce_max(e0.elapsed_time(e1), world, dev), Ks, labels

    xf = torch.from_numpy(emb).to(dev)
    single_ms, K1, lab1 = timed(fms.Context(local), xf)
    ctx = fms.Context(local)
    lo, hi = enable_pixel_sharding(ctx, n)
    xs = xf[lo:hi].contiguous()
    sharded_ms, KN, labN = timed(ctx, xs)
    same = bool(torch.equal(labN[0], lab1[0, lo:hi])) and K1 == KN
    same = reduce_max(0.0 if same else 1.0, world, dev) == 0.0
    return {"config": f"C5: {T} x 512x512 stack, 16-D, 30 tracks, joint clustering ({n} px)", "frames_per_step": T,
            "n_gpus": world, "value": steps * T / (sharded_ms / 1e3), "unit": "frames/s", "scaling": "strong",
            "one_rank_value": steps * T / (single_ms / 1e3), "equal_to_one_rank": same}


def run_reference(args, world, rank):
    if rank != 0:  # the reference arm runs on rank 0 only; other ranks exit 0 without work
        return
    import synth
    f0 = synth.make_frame(args.config, 0)
    # each step clusters one frame of the GPU arm's pool (generator seeds 0, 1, ...), warm-up first
    if args.warmup > 0:
        cpu_run(args.config, 0, 0.0, os.cpu_count() or 1)
    t0 = time.perf_counter()
    runs = [cpu_run(args.config, k, 0.0, os.cpu_count() or 1) for k in range(args.steps)]
    dt = time.perf_counter() - t0
    frames_done = sum(r["frames"] for r in runs)
    secs = sum(r["seconds"] for r in runs)
    cb = {"value": frames_done / secs, "unit": "frames/s", "cores": runs[0]["threads"], "kind": "oracle",
          "sample": f"{args.config} frames of the GPU pool, generator seeds 0..{args.steps - 1}, one per step",
          "seed_iters_per_s": sum(r["seed_iters"] for r in runs) / secs, "cpu_model": cpu_model()}
    # the fms arm's metric and workload strings (same config); each step is a bounded sample of it
    line = {"impl": "reference",
            "metric": f"frames/sec ({f0.H}x{f0.W}, {f0.D}-D embeddings) and mean-shift iteration % of roofline",
            "value": cb["value"], "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {f0.H}x{f0.W} frame, {f0.D}-D, {f0.cells} touching/overlapping "
                                   "cells + background, full OSOP (N_initial 128, gamma 0.9, L 2, P 0.99)",
                       "frames_per_step": 1, "sample": "one frame of the workload per step"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import numpy as np
    import torch

    import paper_2007_14283_b200 as fms
    import synth

    local = local % torch.cuda.device_count()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    B = args.batch
    sharded = args.shard == "seeds" and world > 1
    # pool of 2 batches (inputs 2 x B x 16 MiB > 126 MB L2 for B >= 4), alternated step to step;
    # seed sharding: all ranks work on the same frames
    frames = [synth.make_frame(args.config, 10000 * (0 if sharded else rank) + i) for i in range(2 * B)]
    n, d = frames[0].n, frames[0].D
    pool = torch.from_numpy(np.stack([f.emb for f in frames])).to(dev).view(2, B, n, d)
    euclid = args.metric == "euclid"
    h_run = (2.0 * H) ** 0.5 if euclid else H
    if euclid:  # unit rows: |x - s|^2 = 2 (1 - x.s) at the start, so the windows match cosine h
        pool = pool / pool.norm(dim=-1, keepdim=True)
    labels = torch.empty((B, n), dtype=torch.int32, device=dev)
    cent = torch.empty((B, CAP, d), dtype=torch.float32, device=dev)
    ctx = fms.context(local)
    if sharded:
        from paper_2007_14283_b200.dist import enable_seed_sharding
        enable_seed_sharding(ctx)
    gauss = args.kernel_profile == "gauss"
    if gauss:
        ctx.set_option("kernel_profile", 1)
    if euclid:
        ctx.set_option("metric", 1)
    if args.host_chunk > 0:
        ctx.set_option("host_chunk", args.host_chunk)
    if args.fuse_step:
        ctx.set_option("fuse_step", args.fuse_step)
    if args.no_pdl:
        ctx.set_option("pdl", 0)
    pol = fms.default_policy(**policy_kwargs(n))
    stream = torch.cuda.current_stream(dev)

    def step(k, profile=False):
        rc, K, fs, rs = ctx.cluster_batch_ptr(pool[k % 2].data_ptr(), B, n, d, labels.data_ptr(), cent.data_ptr(),
                                              CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
        return fs, rs

    for k in range(args.warmup):
        step(k)
    totals = dict(iter_ms=0.0, iter_seed_iters=0, iter_count_units=0, iter_launches=0, launches=0, frames=0,
                  seed_iters=0, assign_pairs=0)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # the headline: K steps, no per-kernel instrumentation inside the timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for k in range(args.steps):
            fs, rs = step(k)
            totals["launches"] += rs["launches"]
            totals["frames"] += B
            totals["seed_iters"] += sum(f["seed_iters"] for f in fs)
            totals["assign_pairs"] += sum(sum(f["round_Kc"][:f["rounds"]]) for f in fs)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = reduce_max(ev0.elapsed_time(ev1), world, dev)
    frames_total = totals["frames"] * (1 if sharded else world)
    value = frames_total / (ms / 1e3)
    # a separate profiled pass for the roofline: CUDA events around every K2 launch on the work stream
    prof_steps = max(1, min(args.steps, 6))
    ctx.set_option("profile_iter", 1)
    prof_ms_total = 0.0
    PHASES = ("ms_prep", "ms_select", "ms_step_ctl", "ms_merge", "ms_assign", "ms_host_wait")
    phase_ms = {key: 0.0 for key in PHASES}
    for k in range(prof_steps):
        e0p, e1p = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0p.record(stream)
        fs, rs = step(k)
        e1p.record(stream)
        torch.cuda.synchronize()
        prof_ms_total += e0p.elapsed_time(e1p)
        totals["iter_ms"] += rs["iter_ms"]
        totals["iter_seed_iters"] += rs["iter_seed_iters"]
        totals["iter_count_units"] += rs["iter_count_units"]
        totals["iter_launches"] += rs["iter_launches"]
        for key in PHASES:
            phase_ms[key] += rs[key]
    ctx.set_option("profile_iter", 0)
    # guard pairs: one step with the counting K2 instantiation -- the lockstep window
    # decisions within the similarity's certified error bound of tau (not certified against the
    # exact similarity), per frame and as a fraction of the pairs evaluated
    ctx.set_option("guard_stats", 1)
    gfs, grs = step(0)
    ctx.set_option("guard_stats", 0)
    g_pairs_eval = sum(f["seed_iters"] for f in gfs) * n
    guard = {"per_frame": grs["guard_pairs"] / B, "fraction_of_pairs": grs["guard_pairs"] / max(1, g_pairs_eval),
             "eps": 2.0 ** -16, "frames": B}

    # end-to-end through the host-pointer C-ABI entry (H2D + cluster + D2H inside the call)
    e2e = None
    if not args.no_e2e:
        eh = pool[0].cpu().pin_memory()  # the first input batch (row-normalised for --metric euclid)
        lh = torch.empty((B, n), dtype=torch.int32).pin_memory()
        ch = torch.empty((B, CAP, d), dtype=torch.float32).pin_memory()
        ctx.cluster_host(eh, lh, ch, CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ksteps = max(1, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ksteps):
            ctx.cluster_host(eh, lh, ch, CAP, h_run, MAX_ITERS, None, pol, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = reduce_max(e0.elapsed_time(e1), world, dev)
        e2e = {"value": ksteps * B * (1 if sharded else world) / (ems / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": B * n * d * 4, "d2h_bytes_per_step": B * n * 4 + B * CAP * d * 4}

    peaks, src = measured_peaks()
    # algorithmic: 4 n D per active seed-iteration (similarity + weighted sum) and 2 n D
    # per converged mode in K2's intensity pass (similarity only, R10)
    flops = totals["iter_seed_iters"] * n * 4 * d + totals["iter_count_units"] * n * 2 * d
    achieved = flops / (totals["iter_ms"] / 1e3) / 1e12 if totals["iter_ms"] > 0 else None
    peak = peaks["bf16_tflops_sustained"]
    dp = 16 if d + (2 if euclid else 0) <= 16 else 32  # operand row width of the K2 instantiation
    roof = {"bound": "tensor", "kernel": f"fms::iter8_kernel<{dp}> (K2, int8 exact weighted sum)", "achieved": achieved,
            "peak": peak,
            "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic(),
            "peak_source": f"{src} bf16 dense sustained (fp16 = bf16 rate); burst {peaks['bf16_tflops']}",
            "flops_per_launch": flops / max(1, totals["iter_launches"]),
            "ms_per_launch": totals["iter_ms"] / max(1, totals["iter_launches"]),
            "iter_share_of_step": totals["iter_ms"] / prof_ms_total if prof_ms_total > 0 else None,
            "measured": f"separate profiled pass of {prof_steps} step(s) after the timed region",
            # the rest of the profiled steps by phase (device time per step, host-polled loop)
            "phase_ms_per_step": {"K2": totals["iter_ms"] / prof_steps,
                                  **{k[3:]: v / prof_steps for k, v in phase_ms.items()}}}
    # frame-level roofline: algorithmic iteration FLOPs of the whole timed job at the tensor peak (the
    # K2 launches' work of the timed steps: seed-iterations of every frame)
    job_iter_flops = totals["seed_iters"] * n * 4 * d
    frame_roof_ms = job_iter_flops / (peak * 1e12) * 1e3
    # + the assignment's contraction (2 n D per pixel-centre pair per round) for the job terms
    job_flops = job_iter_flops + totals["assign_pairs"] * n * 2 * d
    job_tensor_ms = job_flops / (peak * 1e12) * 1e3
    # north_star / SURVEY 8(d): the job's roofline is the slowest of three limits -- contraction FLOPs
    # at the tensor peak, kernel exponentials at the SFU peak (0: the flat kernel has none, Eq. 3/11),
    # and embedding bytes at HBM bandwidth (read the fp32 input once, write labels)
    job_frames = totals["frames"]
    hbm_bytes = job_frames * (n * d * 4 + n * 4)
    hbm_ms = hbm_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    roof_terms = {"tensor_ms": job_tensor_ms, "sfu_ms": 0.0, "hbm_ms": hbm_ms,
                  "bound": "tensor" if job_tensor_ms >= hbm_ms else "hbm",
                  "frac": max(job_tensor_ms, hbm_ms) / ms if ms > 0 else None,
                  "hbm_peak_gbs": peaks["hbm_gbs"]}
    # SFU term: the Gaussian profile evaluates one exp2 (MUFU.EX2) per (active seed, pixel) pair of
    # the iteration steps; peak = 148 SMs x 16 MUFU results/clk/SM x the max SM clock (DESIGN 6)
    clk_ghz = (peaks.get("sm_max_mhz") or 1965.0) / 1e3
    sfu_peak = 148 * 16 * clk_ghz  # G exp2/s
    exps = totals["seed_iters"] * n if gauss else 0
    sfu_ms = exps / (sfu_peak * 1e9) * 1e3
    if gauss:
        roof_terms["sfu_ms"] = sfu_ms
        roof_terms["sfu_peak_gexp2_s"] = sfu_peak
        if sfu_ms > max(job_tensor_ms, hbm_ms):
            roof_terms["bound"] = "sfu"
            roof_terms["frac"] = sfu_ms / ms if ms > 0 else None
        ach = totals["iter_seed_iters"] * n / (totals["iter_ms"] / 1e3) / 1e9 if totals["iter_ms"] > 0 else None
        roof = {"bound": "sfu", "kernel": f"fms::iter_kernel<{dp}, true> (K2, Gaussian profile)", "achieved": ach,
                "peak": sfu_peak, "unit": "Gexp2/s", "frac": (ach / sfu_peak) if ach else None, "traffic": None,
                "peak_source": "derived: 148 SMs x 16 MUFU.EX2/clk/SM x sm_max_mhz",
                "tensor_achieved_tflops": achieved, "tensor_peak_tflops": peak,
                "ms_per_launch": totals["iter_ms"] / max(1, totals["iter_launches"]),
                "iter_share_of_step": totals["iter_ms"] / prof_ms_total if prof_ms_total > 0 else None}
    extras = {}
    if world == 1 and not sharded:
        extras = latency_and_b16(ctx, pool, pol, h_run, stream)
        if args.config == CONFIG and not args.no_seed_shard and not gauss and not euclid:
            extras["seed_sharded"] = seed_sharded_c4(1, 0, local)
    cb = None
    if world == 1 and not args.no_cpu:
        cb = cpu_baseline(args.config, budget_s=args.cpu_budget_s)
        cb["gpu_seed_iters_per_s"] = totals["seed_iters"] / (ms / 1e3)
    f0 = frames[0]
    line = {
        "metric": f"frames/sec ({f0.H}x{f0.W}, {d}-D embeddings) and mean-shift iteration % of roofline",
        "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f16x3 split / f32 accumulate (similarity), "
                 + ("f16 weights x f16 limbs -> f32 (weighted sum)" if gauss else "u8 x s8 -> s32 exact (weighted sum)"), "data": "synthetic",
        "config": {"workload": f"{args.config}: {f0.H}x{f0.W} frame, {d}-D, {f0.cells} touching/overlapping cells "
                               f"+ background, full OSOP (N_initial 128, gamma 0.9, L 2, P 0.99)"
                               + (", Gaussian kernel profile (NEXT-4)" if gauss else "")
                               + (", Euclidean metric, rows normalised, h = sqrt(0.2) (NEXT-4)" if euclid else ""),
                   "frames_per_step": B, "l2": "2 alternating input batches of B x 16 MiB (> 126 MB L2)",
                   "parallelism": f"seed-sharded x{world} ({args.backend})" if sharded else f"replicas x{world}"},
        "roofline": roof,
        "guard_pairs": guard,
        "frame_level_frac": frame_roof_ms / ms if ms > 0 else None,
        "job_roofline": roof_terms,
        "seed_iters_per_frame": totals["seed_iters"] / max(1, totals["frames"]),
        "gpu_launches": totals["launches"],
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cb,
    }
    line.update(extras)
    if world > 1 and not sharded and not args.no_seed_shard:
        # strong-scaling extras (C4 seed-sharded, C5 pixel-sharded) after the headline measurement; a
        # watchdog prints the headline line and ends every rank if they overrun (a stuck collective
        # must not cost the run its line)
        import threading

        def _overrun():
            if rank == 0:
                line["sharded_extras"] = "skipped: exceeded the time budget"
                print(json.dumps(line), flush=True)
            os._exit(0)
        guard = threading.Timer(args.extras_budget_s, _overrun)
        guard.daemon = True
        guard.start()
        for key, fn in (("seed_sharded", seed_sharded_c4), ("pixel_sharded", pixel_sharded_c5)):
            try:
                line[key] = fn(world, rank, local)
            except Exception as e:  # reported, not fatal: the replicas line is the headline
                line[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
        guard.cancel()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
