"""fp64 CPU oracle of Faster Mean-shift (ctypes wrapper around fms_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "fms_oracle.c")

SEEDS_FIXED, SEEDS_OSOP, SEEDS_ALL = 0, 1, 2
MAX_ROUNDS = 16
OK, E_INVALID, E_ZERO_NORM, E_STALLED, E_CAPACITY = 0, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, OpenMP over seeds/pixels).  No FMA contraction, so the
    arithmetic is exactly the source's."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "fms_oracle.h"))):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_seeds", C.c_int32), ("gamma", C.c_double),
                ("L", C.c_double), ("H", C.c_double), ("P", C.c_double),
                ("has_background", C.c_int32), ("min_instance_px", C.c_int32),
                ("saturation_stop", C.c_int32), ("max_rounds", C.c_int32),
                ("rng_seed", C.c_uint64), ("profile", C.c_int32), ("metric", C.c_int32)]


PROFILE_FLAT, PROFILE_GAUSS = 0, 1
METRIC_COSINE, METRIC_EUCLID = 0, 1


class Trace(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("K", C.c_int32), ("seeds_total", C.c_int64),
                ("seed_iters", C.c_int64), ("discarded", C.c_int64),
                ("round_K", C.c_int32 * MAX_ROUNDS), ("round_iters", C.c_int32 * MAX_ROUNDS),
                ("round_conv", C.c_int32 * MAX_ROUNDS), ("round_disc", C.c_int32 * MAX_ROUNDS),
                ("round_seed_iters", C.c_int64 * MAX_ROUNDS),
                ("round_Kc", C.c_int32 * MAX_ROUNDS), ("round_I", C.c_int32 * MAX_ROUNDS),
                ("round_cand", C.c_int64 * MAX_ROUNDS), ("round_r", C.c_double * MAX_ROUNDS),
                ("round_nmin", C.c_double * MAX_ROUNDS)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = np.ctypeslib.ndpointer
        L.fmso_splitmix64.restype = C.c_uint64
        L.fmso_splitmix64.argtypes = [C.c_uint64]
        L.fmso_key.restype = C.c_uint64
        L.fmso_key.argtypes = [C.c_uint64, C.c_int32, C.c_int64]
        L.fmso_p_success.restype = C.c_double
        L.fmso_p_success.argtypes = [C.c_int64, C.c_int64, C.c_double]
        L.fmso_n_min.restype = C.c_int64
        L.fmso_n_min.argtypes = [C.c_double, C.c_int64, C.c_double]
        L.fmso_session_next.restype = C.c_int64
        L.fmso_session_next.argtypes = [C.c_int64, C.c_double, C.c_double]
        L.fmso_need.restype = C.c_int32
        L.fmso_need.argtypes = [C.c_double, C.c_int64]
        L.fmso_normalize.restype = C.c_int
        L.fmso_normalize.argtypes = [P(np.float32, flags="C"), C.c_int64, C.c_int32, P(np.float64, flags="C")]
        L.fmso_select.restype = C.c_int64
        L.fmso_select.argtypes = [P(np.uint8, flags="C"), C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                  P(np.int64, flags="C")]
        L.fmso_window.restype = C.c_int64
        L.fmso_window.argtypes = [P(np.float64, flags="C"), C.c_int64, C.c_int32, C.c_double,
                                  P(np.float64, flags="C"), P(np.float64, flags="C")]
        L.fmso_lockstep.restype = C.c_int32
        L.fmso_lockstep.argtypes = [P(np.float64, flags="C"), C.c_int64, C.c_int32, C.c_double, C.c_int32,
                                    C.c_double, C.c_double, C.c_int64, P(np.float64, flags="C"),
                                    P(np.uint8, flags="C"), P(np.int64, flags="C"), P(np.int32, flags="C"),
                                    C.POINTER(C.c_int64)]
        L.fmso_lockstep_p.restype = C.c_int32
        L.fmso_lockstep_p.argtypes = L.fmso_lockstep.argtypes + [C.c_int32]
        L.fmso_window_gauss.restype = C.c_double
        L.fmso_window_gauss.argtypes = [P(np.float64, flags="C"), C.c_int64, C.c_int32, C.c_double,
                                        P(np.float64, flags="C"), P(np.float64, flags="C")]
        L.fmso_merge.restype = C.c_int64
        L.fmso_merge.argtypes = [P(np.float64, flags="C"), P(np.int64, flags="C"), P(np.int64, flags="C"),
                                 C.c_int64, C.c_int32, C.c_double, P(np.int64, flags="C")]
        L.fmso_assign.restype = None
        L.fmso_assign.argtypes = [P(np.float64, flags="C"), C.c_int64, C.c_int32, P(np.float64, flags="C"),
                                  C.c_int64, C.c_double, P(np.int32, flags="C"), P(np.uint8, flags="C"),
                                  P(np.int64, flags="C")]
        L.fmso_cluster.restype = C.c_int
        L.fmso_cluster.argtypes = [P(np.float32, flags="C"), C.c_int64, C.c_int32, C.c_double, C.c_int32,
                                   C.c_double, C.POINTER(Policy), P(np.int32, flags="C"),
                                   P(np.float64, flags="C"), C.c_int32, C.POINTER(C.c_int32),
                                   C.POINTER(Trace)]
        L.fmso_num_threads.restype = C.c_int
        L.fmso_observe.restype = C.c_int64
        L.fmso_observe.argtypes = [P(np.int64, flags="C"), C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.fmso_osop_stop.restype = C.c_int
        L.fmso_osop_stop.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64,
                                     C.c_double, C.c_int32, C.c_int32, C.c_int32]
        _lib = L
    return _lib


def policy(kind=SEEDS_OSOP, n_seeds=128, gamma=0.9, L=2.0, H=8.0, P=0.99, has_background=1,
           min_instance_px=0, saturation_stop=0, max_rounds=8, rng_seed=0, profile=PROFILE_FLAT,
           metric=METRIC_COSINE) -> Policy:
    return Policy(kind, n_seeds, gamma, L, H, P, has_background, min_instance_px, saturation_stop,
                  max_rounds, rng_seed, profile, metric)


@dataclass
class Result:
    status: int
    labels: np.ndarray
    centres: np.ndarray
    K: int
    trace: dict = field(default_factory=dict)


def trace_dict(tr: Trace) -> dict:
    R = tr.rounds
    return dict(rounds=R, K=tr.K, seeds_total=tr.seeds_total, seed_iters=tr.seed_iters,
                discarded=tr.discarded, round_K=list(tr.round_K[:R]), round_iters=list(tr.round_iters[:R]),
                round_conv=list(tr.round_conv[:R]), round_disc=list(tr.round_disc[:R]),
                round_seed_iters=list(tr.round_seed_iters[:R]), round_Kc=list(tr.round_Kc[:R]),
                round_I=list(tr.round_I[:R]), round_cand=list(tr.round_cand[:R]),
                round_r=list(tr.round_r[:R]), round_nmin=list(tr.round_nmin[:R]))


def cluster(emb: np.ndarray, h: float = 0.1, max_iter: int = 300, tol: float | None = None,
            pol: Policy | None = None, centres_cap: int = 65536) -> Result:
    emb = np.ascontiguousarray(emb, dtype=np.float32)
    n, d = emb.shape
    tol = h / 1000.0 if tol is None else tol
    pol = pol if pol is not None else policy()
    labels = np.zeros(n, dtype=np.int32)
    centres = np.zeros((centres_cap, d), dtype=np.float64)
    K = C.c_int32(0)
    tr = Trace()
    rc = lib().fmso_cluster(emb, n, d, h, max_iter, tol, C.byref(pol), labels, centres, centres_cap,
                            C.byref(K), C.byref(tr))
    return Result(rc, labels, centres[:K.value].copy(), K.value, trace_dict(tr))


def normalize(emb: np.ndarray) -> np.ndarray:
    emb = np.ascontiguousarray(emb, dtype=np.float32)
    out = np.zeros(emb.shape, dtype=np.float64)
    rc = lib().fmso_normalize(emb, emb.shape[0], emb.shape[1], out)
    if rc != OK:
        raise ValueError(f"normalize failed: {rc}")
    return out


def select(cand: np.ndarray, K: int, rng_seed: int, round_: int) -> np.ndarray:
    cand = np.ascontiguousarray(cand, dtype=np.uint8)
    out = np.zeros(max(1, int(cand.sum())), dtype=np.int64)
    k = lib().fmso_select(cand, cand.size, K, rng_seed, round_, out)
    return out[:k].copy()


def window(xhat: np.ndarray, s: np.ndarray, h: float):
    g = np.zeros(xhat.shape[1], dtype=np.float64)
    cnt = lib().fmso_window(np.ascontiguousarray(xhat), xhat.shape[0], xhat.shape[1], 1.0 - h,
                            np.ascontiguousarray(s, dtype=np.float64), g)
    return g, int(cnt)


def window_gauss(xhat: np.ndarray, s: np.ndarray, h: float):
    g = np.zeros(xhat.shape[1], dtype=np.float64)
    mass = lib().fmso_window_gauss(np.ascontiguousarray(xhat), xhat.shape[0], xhat.shape[1], h,
                                   np.ascontiguousarray(s, dtype=np.float64), g)
    return g, float(mass)


def lockstep(xhat: np.ndarray, seeds: np.ndarray, h: float, max_iter: int = 300, tol: float | None = None,
             gamma: float = 0.9, profile: int = PROFILE_FLAT):
    xhat = np.ascontiguousarray(xhat, dtype=np.float64)
    s = np.ascontiguousarray(seeds, dtype=np.float64).copy()
    K = s.shape[0]
    st = np.zeros(K, dtype=np.uint8)
    inten = np.zeros(K, dtype=np.int64)
    its = np.zeros(K, dtype=np.int32)
    sit = C.c_int64(0)
    tol = h / 1000.0 if tol is None else tol
    t = lib().fmso_lockstep_p(xhat, xhat.shape[0], xhat.shape[1], h, max_iter, tol, gamma, K, s, st, inten,
                              its, C.byref(sit), profile)
    return dict(iters=int(t), seeds=s, status=st, intensity=inten, seed_iters_each=its, seed_iters=sit.value)


def merge(pool: np.ndarray, intensity: np.ndarray, origin: np.ndarray, rho: float) -> np.ndarray:
    m, d = pool.shape
    keep = np.zeros(max(1, m), dtype=np.int64)
    k = lib().fmso_merge(np.ascontiguousarray(pool, dtype=np.float64),
                         np.ascontiguousarray(intensity, dtype=np.int64),
                         np.ascontiguousarray(origin, dtype=np.int64), m, d, rho, keep)
    return keep[:k].copy()


def assign(xhat: np.ndarray, centres: np.ndarray, h: float):
    n, d = xhat.shape
    K = centres.shape[0]
    labels = np.zeros(n, dtype=np.int32)
    cov = np.zeros(n, dtype=np.uint8)
    hist = np.zeros(max(1, K), dtype=np.int64)
    lib().fmso_assign(np.ascontiguousarray(xhat), n, d, np.ascontiguousarray(centres, dtype=np.float64), K,
                      1.0 - h, labels, cov, hist)
    return labels, cov, hist[:K]


def p_success(N: int, I: int, r: float) -> float:
    return lib().fmso_p_success(N, I, r)


def n_min(P: float, I: int, r: float) -> int:
    return lib().fmso_n_min(P, I, r)


def session_next(total: int, nmin: float, H: float) -> int:
    """O8: seed count carried to the next frame (R12, R18); nmin < 0 = infinite."""
    return lib().fmso_session_next(int(total), float(nmin), float(H))


def session(frames, h: float = 0.1, max_iter: int = 300, tol: float | None = None, pol: Policy | None = None,
            centres_cap: int = 65536):
    """NEXT-1: cluster a frame sequence, carrying the OSOP seed count N across frames (O8): frame
    t's round 0 uses N_t seeds; N_{t+1} = session_next(seeds used by frame t, its last N_min, H).
    Returns (results, N sequence)."""
    pol = pol if pol is not None else policy()
    N = int(pol.n_seeds)
    out, Ns = [], []
    for emb in frames:
        p = policy(pol.kind, N, pol.gamma, pol.L, pol.H, pol.P, pol.has_background, pol.min_instance_px,
                   pol.saturation_stop, pol.max_rounds, pol.rng_seed, pol.profile, pol.metric)
        r = cluster(emb, h=h, max_iter=max_iter, tol=tol, pol=p, centres_cap=centres_cap)
        out.append(r)
        Ns.append(N)
        if r.status != 0:
            break
        nm = r.trace["round_nmin"][-1] if r.trace["rounds"] > 0 else -1.0
        N = max(1, session_next(r.trace["seeds_total"], nm, pol.H))
    return out, Ns


def observe(hist, n: int, has_background: int = 1, min_instance_px: int = 0):
    """OSOP observation (R14, R22): returns (background index or -1, I, r)."""
    hist = np.ascontiguousarray(hist, dtype=np.int64)
    I = C.c_int32(0)
    r = C.c_double(0.0)
    bg = lib().fmso_observe(hist if hist.size else np.zeros(1, np.int64), hist.size, int(n), int(has_background),
                            int(min_instance_px), C.byref(I), C.byref(r))
    return int(bg), I.value, r.value


NMIN_INF = 2 ** 63 - 1


def osop_stop(ncand: int, total: int, n: int, round_: int, max_rounds: int, nmin: int, L: float,
              saturation_stop: int, I: int, I_prev: int) -> bool:
    """OSOP stop rule after a round (R13, R22); nmin = NMIN_INF is infinite."""
    return bool(lib().fmso_osop_stop(ncand, total, n, round_, max_rounds, nmin, L, saturation_stop, I, I_prev))


def key(rng_seed: int, round_: int, i: int) -> int:
    return lib().fmso_key(rng_seed, round_, i)
