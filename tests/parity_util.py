"""Comparison helpers for CUDA-vs-oracle parity (test-only)."""
import numpy as np
from scipy.optimize import linear_sum_assignment
from sklearn.metrics import adjusted_rand_score


def bijection(a, b) -> bool:
    """Two labelings are the same partition (contingency table: one nonzero per row and column)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    pairs = np.unique(a.astype(np.int64) * (1 << 32) + b.astype(np.int64))
    return pairs.size == np.unique(a).size == np.unique(b).size


def match_centres(cg: np.ndarray, co: np.ndarray):
    """Hungarian matching on cosine distance; returns (rows, cols, distances)."""
    cg = cg / np.linalg.norm(cg, axis=1, keepdims=True)
    co = co / np.linalg.norm(co, axis=1, keepdims=True)
    D = 1.0 - cg.astype(np.float64) @ co.astype(np.float64).T
    r, c = linear_sum_assignment(D)
    return r, c, D[r, c]


def ari(a, b) -> float:
    return float(adjusted_rand_score(np.asarray(a).ravel(), np.asarray(b).ravel()))
