"""Python binding of libfms.so, the B200 (sm_100a) Faster Mean-shift hot path.

Argument marshalling only: every step of the method runs in the CUDA kernels behind the C ABI
(include/fms.h).  There is no CPU or PyTorch fallback: if the library is missing or no sm_100
device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

SEEDS_FIXED, SEEDS_OSOP, SEEDS_ALL = 0, 1, 2
MAX_ROUNDS = 16
STATUS = {0: "OK", 2: "INVALID", 3: "ZERO_NORM", 4: "STALLED", 5: "CAPACITY", 6: "CUDA", 7: "NCCL", 8: "OOM",
          9: "INTERNAL"}
EXPORTS = ["fms_default_policy", "fms_ctx_create", "fms_ctx_destroy", "fms_last_error", "fms_version",
           "fms_set_option", "fms_set_exchange", "fms_set_pixel_shard", "fms_cluster", "fms_cluster_batch", "fms_cluster_batch_host",
           "fms_session_create", "fms_session_step", "fms_session_seeds", "fms_session_destroy",
           "fms_set_allgather", "fms_nccl_unique_id", "fms_set_nccl", "fms_ctx_create_dist"]
SHARD_SEEDS, SHARD_PIXELS = 1, 2

# int (*)(void* user, int32_t* buf, int64_t count, void* stream): in-place int32 sum over ranks
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
# int (*)(void* user, const int32_t* send, int32_t* recv, int64_t count, void* stream): all-gather
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfms.so")


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_seeds", C.c_int32), ("gamma", C.c_double), ("L", C.c_double),
                ("H", C.c_double), ("P", C.c_double), ("has_background", C.c_int32),
                ("min_instance_px", C.c_int32), ("saturation_stop", C.c_int32), ("max_rounds", C.c_int32),
                ("rng_seed", C.c_uint64)]


class FrameStats(C.Structure):
    _fields_ = [("status", C.c_int32), ("rounds", C.c_int32), ("K", C.c_int32), ("pad", C.c_int32),
                ("seeds_total", C.c_int64), ("seed_iters", C.c_int64), ("discarded", C.c_int64),
                ("round_K", C.c_int32 * MAX_ROUNDS), ("round_iters", C.c_int32 * MAX_ROUNDS),
                ("round_conv", C.c_int32 * MAX_ROUNDS), ("round_disc", C.c_int32 * MAX_ROUNDS),
                ("round_Kc", C.c_int32 * MAX_ROUNDS), ("round_I", C.c_int32 * MAX_ROUNDS),
                ("round_seed_iters", C.c_int64 * MAX_ROUNDS), ("round_cand", C.c_int64 * MAX_ROUNDS),
                ("round_r", C.c_double * MAX_ROUNDS), ("round_nmin", C.c_double * MAX_ROUNDS)]

    def as_dict(self) -> dict:
        R = self.rounds
        return dict(status=self.status, rounds=R, K=self.K, seeds_total=self.seeds_total,
                    seed_iters=self.seed_iters, discarded=self.discarded,
                    round_K=list(self.round_K[:R]), round_iters=list(self.round_iters[:R]),
                    round_conv=list(self.round_conv[:R]), round_disc=list(self.round_disc[:R]),
                    round_seed_iters=list(self.round_seed_iters[:R]), round_Kc=list(self.round_Kc[:R]),
                    round_I=list(self.round_I[:R]), round_cand=list(self.round_cand[:R]),
                    round_r=list(self.round_r[:R]), round_nmin=list(self.round_nmin[:R]))


class RunStats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("workspace_bytes", C.c_int64), ("steps", C.c_int32),
                ("iter_launches", C.c_int32), ("iter_ms", C.c_double), ("iter_seed_iters", C.c_int64),
                ("iter_items", C.c_int64), ("launches", C.c_int64), ("iter_count_units", C.c_int64),
                ("host_syncs", C.c_int64), ("ms_prep", C.c_double), ("ms_select", C.c_double),
                ("ms_step_ctl", C.c_double), ("ms_merge", C.c_double), ("ms_assign", C.c_double),
                ("ms_host_wait", C.c_double), ("guard_pairs", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    """Load libfms.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2007_14283_b200.build` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.fms_version.restype = C.c_char_p
        L.fms_last_error.restype = C.c_char_p
        L.fms_last_error.argtypes = [vp]
        L.fms_default_policy.argtypes = [C.POINTER(Policy)]
        L.fms_ctx_create.argtypes = [C.POINTER(vp), C.c_int]
        L.fms_ctx_destroy.argtypes = [vp]
        L.fms_ctx_destroy.restype = None
        L.fms_set_option.argtypes = [vp, C.c_char_p, i64]
        L.fms_set_exchange.argtypes = [vp, EXCHANGE_FN, vp, i32, i32]
        L.fms_set_pixel_shard.argtypes = [vp, EXCHANGE_FN, vp, i32, i32, i64, i64]
        L.fms_set_allgather.argtypes = [vp, ALLGATHER_FN, vp]
        L.fms_nccl_unique_id.argtypes = [vp]
        L.fms_set_nccl.argtypes = [vp, vp, i32, i32, i32, i64, i64]
        L.fms_ctx_create_dist.argtypes = [C.POINTER(vp), C.c_int, vp, i32, i32, i32, i64, i64]
        L.fms_session_create.argtypes = [vp, C.POINTER(Policy), C.POINTER(vp)]
        L.fms_session_create.restype = C.c_int
        L.fms_session_step.argtypes = [vp, vp, i64, i32] + [f64, i32, f64, vp, vp, i32, vp, vp, C.POINTER(RunStats), vp]
        L.fms_session_step.restype = C.c_int
        L.fms_session_seeds.argtypes = [vp]
        L.fms_session_seeds.restype = i64
        L.fms_session_destroy.argtypes = [vp]
        L.fms_session_destroy.restype = None
        common = [f64, i32, f64, C.POINTER(Policy), vp, vp, i32, vp, vp, C.POINTER(RunStats), vp]
        L.fms_cluster.argtypes = [vp, vp, i64, i32] + common
        L.fms_cluster_batch.argtypes = [vp, vp, i32, i64, i32] + common
        L.fms_cluster_batch_host.argtypes = [vp, vp, i32, i64, i32] + common
        for fn in ("fms_default_policy", "fms_ctx_create", "fms_set_option", "fms_set_exchange",
                   "fms_set_pixel_shard", "fms_set_allgather", "fms_nccl_unique_id", "fms_set_nccl",
                   "fms_ctx_create_dist", "fms_cluster",
                   "fms_cluster_batch", "fms_cluster_batch_host"):
            getattr(L, fn).restype = C.c_int
        _lib = L
    return _lib


def default_policy(**kw) -> Policy:
    p = Policy()
    lib().fms_default_policy(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class FmsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"fms status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class Context:
    """One fms context (device workspace, TMA descriptors) on one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        rc = lib().fms_ctx_create(C.byref(h), device)
        if rc != 0:
            raise FmsError(rc, f"fms_ctx_create(device={device}) failed (needs an sm_100 GPU)")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().fms_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        self._check(lib().fms_set_option(self.h, key.encode(), int(value)))

    def set_exchange(self, fn, rank: int, world: int):
        """Seed sharding (include/fms.h fms_set_exchange).  fn(buf_ptr, count, stream_ptr) must replace
        the int32 device buffer by its sum over all ranks, ordered on the given stream, and return 0;
        world = 1 (fn None) turns sharding off.  paper_2007_14283_b200.dist builds fn from
        torch.distributed."""
        self._xfn = self._wrap_exchange(fn)  # kept alive with the context
        self._check(lib().fms_set_exchange(self.h, self._xfn, None, int(rank), int(world)))

    def _wrap_exchange(self, fn):
        if fn is None:
            return EXCHANGE_FN()

        def _cb(user, buf, count, stream, _fn=fn):
            try:
                return int(_fn(buf, count, stream or 0))
            except Exception as e:  # a Python exception must not unwind through the C library
                self._xerr = e
                return 1
        return EXCHANGE_FN(_cb)

    def set_allgather(self, fn):
        """Seed sharding's round exchange as an all-gather (include/fms.h fms_set_allgather):
        fn(send_ptr, recv_ptr, count, stream_ptr) gathers every rank's `count` int32 values into recv
        (rank order), ordered on the stream; None restores the all-reduce exchange."""
        if fn is None:
            self._gfn = ALLGATHER_FN()
        else:
            def _cb(user, send, recv, count, stream, _fn=fn):
                try:
                    return int(_fn(send, recv, count, stream or 0))
                except Exception as e:  # must not unwind through the C library
                    self._xerr = e
                    return 1
            self._gfn = ALLGATHER_FN(_cb)
        self._check(lib().fms_set_allgather(self.h, self._gfn, None))

    def set_nccl(self, unique_id: bytes, rank: int, world: int, mode: int, n_global: int = 0, offset: int = 0):
        """In-library NCCL sharding (include/fms.h fms_set_nccl); unique_id = the 128 bytes of
        nccl_unique_id() from rank 0.  Collective over the `world` ranks."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(lib().fms_set_nccl(self.h, buf, int(rank), int(world), int(mode), int(n_global), int(offset)))

    def set_pixel_shard(self, fn, rank: int, world: int, n_global: int, offset: int):
        """Pixel sharding (include/fms.h fms_set_pixel_shard): this rank holds pixels
        [offset, offset + n) of frames of n_global pixels; fn as in set_exchange."""
        self._pfn = self._wrap_exchange(fn)  # kept alive with the context
        self._check(lib().fms_set_pixel_shard(self.h, self._pfn, None, int(rank), int(world), int(n_global),
                                              int(offset)))

    def _check(self, rc: int, allow=()):
        if rc != 0 and rc not in allow:
            raise FmsError(rc, lib().fms_last_error(self.h).decode())
        return rc

    def cluster_batch_ptr(self, emb_ptr: int, B: int, n: int, d: int, labels_ptr: int, centres_ptr: int,
                          centres_cap: int, h: float = 0.1, max_iters: int = 300, tol: float | None = None,
                          policy: Policy | None = None, stream: int = 0, allow=()):
        """Raw-pointer entry (device pointers).  Returns (status, K[B], frame stats, run stats)."""
        tol = h / 1000.0 if tol is None else tol
        policy = policy if policy is not None else default_policy()
        K = (C.c_int32 * B)()
        fs = (FrameStats * B)()
        rs = RunStats()
        rc = lib().fms_cluster_batch(self.h, C.c_void_p(emb_ptr), B, n, d, h, max_iters, tol, C.byref(policy),
                                     C.c_void_p(labels_ptr), C.c_void_p(centres_ptr), centres_cap, K, fs,
                                     C.byref(rs), C.c_void_p(stream))
        self._check(rc, allow)
        return rc, list(K), [f.as_dict() for f in fs], rs.as_dict()

    def cluster(self, emb, h: float = 0.1, max_iters: int = 300, tol: float | None = None,
                policy: Policy | None = None, centres_cap: int = 4096, allow=()):
        """emb: torch CUDA float32 tensor [n, d] or [B, n, d].  Returns (labels, centres, K, stats).
        labels: int32 [B, n]; centres: float32 [B, centres_cap, d] (rows < K valid)."""
        import torch
        if emb.dim() == 2:
            emb = emb.unsqueeze(0)
        if not (emb.is_cuda and emb.dtype == torch.float32):
            raise TypeError("emb must be a CUDA float32 tensor")
        emb = emb.contiguous()
        B, n, d = emb.shape
        labels = torch.empty((B, n), dtype=torch.int32, device=emb.device)
        centres = torch.zeros((B, max(centres_cap, 1), d), dtype=torch.float32, device=emb.device)
        stream = torch.cuda.current_stream(emb.device).cuda_stream
        rc, K, fs, rs = self.cluster_batch_ptr(emb.data_ptr(), B, n, d, labels.data_ptr(), centres.data_ptr(),
                                               centres_cap, h, max_iters, tol, policy, stream, allow)
        return labels, centres, K, dict(status=rc, frames=fs, run=rs)

    def cluster_host(self, emb_host, labels_host, centres_host, centres_cap: int, h: float = 0.1,
                     max_iters: int = 300, tol: float | None = None, policy: Policy | None = None, stream: int = 0,
                     allow=()):
        """Host-buffer entry (end-to-end): emb_host [B,n,d] float32, labels_host [B,n] int32,
        centres_host [B,cap,d] float32 -- all contiguous CPU torch tensors (pinned for the copies to
        overlap).  Shapes and dtypes are checked before the call: the library writes B*n labels and
        B*centres_cap*d centre values through the raw pointers."""
        import torch
        for name, t, dt in (("emb_host", emb_host, torch.float32), ("labels_host", labels_host, torch.int32),
                            ("centres_host", centres_host, torch.float32)):
            if not isinstance(t, torch.Tensor):
                raise TypeError(f"{name} must be a torch tensor")
            if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous():
                raise TypeError(f"{name} must be a contiguous CPU {dt} tensor")
        if emb_host.dim() != 3:
            raise ValueError("emb_host must be [B, n, d]")
        B, n, d = emb_host.shape
        if tuple(labels_host.shape) != (B, n):
            raise ValueError(f"labels_host must be [{B}, {n}], got {tuple(labels_host.shape)}")
        if centres_cap < 0 or centres_host.dim() != 3 or centres_host.shape[0] != B or \
                centres_host.shape[1] != centres_cap or centres_host.shape[2] != d:
            raise ValueError(f"centres_host must be [{B}, centres_cap={centres_cap}, {d}], "
                             f"got {tuple(centres_host.shape)}")
        tol = h / 1000.0 if tol is None else tol
        policy = policy if policy is not None else default_policy()
        K = (C.c_int32 * B)()
        rs = RunStats()
        rc = lib().fms_cluster_batch_host(self.h, C.c_void_p(emb_host.data_ptr()), B, n, d, h, max_iters, tol,
                                          C.byref(policy), C.c_void_p(labels_host.data_ptr()),
                                          C.c_void_p(centres_host.data_ptr()), centres_cap, K, None,
                                          C.byref(rs), C.c_void_p(stream))
        self._check(rc, allow)
        return rc, list(K), rs.as_dict()


class Session:
    """NEXT-1 frame sequence (include/fms.h fms_session_*): the OSOP seed count N carries from one
    frame to the next."""

    def __init__(self, ctx: Context, policy: Policy | None = None):
        self.ctx = ctx
        policy = policy if policy is not None else default_policy()
        h = C.c_void_p()
        ctx._check(lib().fms_session_create(ctx.h, C.byref(policy), C.byref(h)))
        self.h = h

    @property
    def seeds(self) -> int:
        """N for round 0 of the next frame."""
        return int(lib().fms_session_seeds(self.h))

    def step(self, emb, h: float = 0.1, max_iters: int = 300, tol: float | None = None, centres_cap: int = 4096,
             allow=()):
        """emb: CUDA float32 [n, d].  Returns (labels [n], centres [cap, d], K, frame stats)."""
        import torch
        if not (emb.is_cuda and emb.dtype == torch.float32 and emb.dim() == 2):
            raise TypeError("emb must be a CUDA float32 tensor [n, d]")
        emb = emb.contiguous()
        n, d = emb.shape
        tol = h / 1000.0 if tol is None else tol
        labels = torch.empty((n,), dtype=torch.int32, device=emb.device)
        centres = torch.zeros((max(centres_cap, 1), d), dtype=torch.float32, device=emb.device)
        K = C.c_int32()
        fs = FrameStats()
        rs = RunStats()
        stream = torch.cuda.current_stream(emb.device).cuda_stream
        rc = lib().fms_session_step(self.h, C.c_void_p(emb.data_ptr()), n, d, h, max_iters, tol,
                                    C.c_void_p(labels.data_ptr()), C.c_void_p(centres.data_ptr()), centres_cap,
                                    C.byref(K), C.byref(fs), C.byref(rs), C.c_void_p(stream))
        self.ctx._check(rc, allow)
        return labels, centres, K.value, fs.as_dict()

    def close(self):
        if getattr(self, "h", None):
            lib().fms_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the library's NCCL (include/fms.h fms_nccl_unique_id)."""
    buf = C.create_string_buffer(128)
    rc = lib().fms_nccl_unique_id(buf)
    if rc != 0:
        raise FmsError(rc, "fms_nccl_unique_id failed (libnccl.so.2 not available?)")
    return buf.raw


_ctxs: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    if device not in _ctxs:
        _ctxs[device] = Context(device)
    return _ctxs[device]


def cluster(emb, h: float = 0.1, max_iters: int = 300, tol: float | None = None, policy: Policy | None = None,
            centres_cap: int = 4096, allow=()):
    """Cluster one frame [n, d] or a batch [B, n, d] of CUDA float32 embeddings (see Context.cluster)."""
    return context(emb.device.index or 0).cluster(emb, h, max_iters, tol, policy, centres_cap, allow)
