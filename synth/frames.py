"""Seeded synthetic cell frames of cosine embeddings (data generation only).

Recipe.  It mirrors the paper's simulations:
a background cluster holding most pixels ("the blue data-set had 750 points,
accounting for 50%"), cluster directions that are "orthogonal or opposite" (signed basis
vectors), and Gaussian noise.  Frame shapes are those of the paper's figures and
cohorts (512x512 in Fig. 1; ISBI frame sizes P:451).

* Frame H x W -> embeddings float32 [H*W, D], row-major, raster pixel order.
* Directions: background mu_0 and one direction per cell.  If #clusters <= 2D they are distinct
  signed basis vectors +-e_j (pairwise cos in {0,-1}); otherwise rejection-sampled unit vectors
  with pairwise cos <= 0.5.
* Geometry: discs with uniform centres and radii drawn from the config's range.
  - "hard": non-touching discs (gap >= `gap` px), one-hot ownership (well-separated frames).
  - "soft": discs may touch/overlap; a later disc is painted over earlier ones with a soft edge
    a_k = sigmoid((R_k - dist)/0.7 px): v <- (1-a_k) v + 4 a_k mu_k (cell weight
    4*sigmoid, the layer below weighted by 1-sigmoid).  Truth = topmost disc with a_k > 1/2.
* Pixel embedding: x = normalize(v/|v| + sigma*eps), eps ~ N(0, I) clipped to +-3, multiplied by a
  per-pixel norm factor U[0.5, 2] so the method's own normalisation (Eq. 1/9) is exercised.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# name -> parameters.  radius in px; sigma = embedding noise; min_px = min_instance_px proposal.
CONFIGS: dict[str, dict] = {
    # C1: BASELINE.json configs[0] (64x64, 5 well-separated cells + background, fixed 64 seeds)
    "C1": dict(H=64, W=64, D=16, cells=5, radius=(10, 12), sigma=0.02, boundary="hard", gap=2),
    # C2: BASELINE.json configs[1] (512x512, ~30 touching/overlapping cells, full OSOP) - the metric
    "C2": dict(H=512, W=512, D=16, cells=30, radius=(20, 35), sigma=0.02, boundary="soft", gap=0),
    # well-separated 512x512 variant (exact-parity case at the metric's frame size)
    "C2sep": dict(H=512, W=512, D=16, cells=30, radius=(20, 30), sigma=0.02, boundary="hard", gap=2),
    # C3: ISBI-shaped cohorts (sizes as printed at P:451; cell counts/radii assumed)
    "C3_hela": dict(H=512, W=512, D=16, cells=40, radius=(25, 35), sigma=0.02, boundary="soft", gap=0),
    "C3_gowt1": dict(H=1024, W=1024, D=16, cells=25, radius=(30, 45), sigma=0.02, boundary="soft", gap=0),
    "C3_simplus": dict(H=520, W=696, D=16, cells=30, radius=(12, 20), sigma=0.02, boundary="soft", gap=0),
    "C3_u373": dict(H=718, W=660, D=16, cells=8, radius=(30, 60), sigma=0.02, boundary="soft", gap=0),
    # C4: 1024x1024, 32-D, ~200 cells (rejection-sampled directions)
    "C4": dict(H=1024, W=1024, D=32, cells=200, radius=(20, 30), sigma=0.02, boundary="soft", gap=0),
    # small soft frame for fast near-boundary parity tests
    "S1": dict(H=128, W=128, D=16, cells=8, radius=(10, 18), sigma=0.02, boundary="soft", gap=0),
    "S1sep": dict(H=128, W=128, D=16, cells=8, radius=(8, 14), sigma=0.02, boundary="hard", gap=2),
    "S32sep": dict(H=96, W=96, D=32, cells=6, radius=(8, 12), sigma=0.02, boundary="hard", gap=2),
}

_CFG_IDS = {name: i for i, name in enumerate(sorted(CONFIGS))}


@dataclass
class Frame:
    emb: np.ndarray      # float32 [n, D]
    truth: np.ndarray    # int32 [n]; 0 = background, k = cell k
    H: int
    W: int
    D: int
    cells: int
    config: str
    seed: int

    @property
    def n(self) -> int:
        return self.H * self.W


def _directions(rng: np.random.Generator, k: int, D: int) -> np.ndarray:
    dirs = np.zeros((k, D), dtype=np.float64)
    if k <= 2 * D:
        order = rng.permutation(2 * D)[:k]
        for t, o in enumerate(order):
            dirs[t, o // 2] = 1.0 if o % 2 == 0 else -1.0
        return dirs
    got = 0
    while got < k:
        v = rng.standard_normal(D)
        v /= np.sqrt(np.sum(v * v))
        if got == 0 or np.max(dirs[:got] @ v) <= 0.5:
            dirs[got] = v
            got += 1
    return dirs


def _discs(rng, cfg, hard: bool):
    H, W, (r0, r1), cells, gap = cfg["H"], cfg["W"], cfg["radius"], cfg["cells"], cfg["gap"]
    for _restart in range(1000):
        out = []
        tries = 0
        while len(out) < cells and tries < 2000 * cells:
            tries += 1
            R = rng.uniform(r0, r1)
            cy = rng.uniform(R + 1, H - R - 1)
            cx = rng.uniform(R + 1, W - R - 1)
            if hard and any((cy - y) ** 2 + (cx - x) ** 2 < (R + r + gap + 1.0) ** 2 for (y, x, r) in out):
                continue
            out.append((cy, cx, R))
        if len(out) == cells:
            return out
    raise RuntimeError("could not place discs")


def make_frame(config: str, seed: int) -> Frame:
    cfg = CONFIGS[config]
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 1000 + _CFG_IDS[config]]))
    H, W, D, cells = cfg["H"], cfg["W"], cfg["D"], cfg["cells"]
    hard = cfg["boundary"] == "hard"
    dirs = _directions(rng, cells + 1, D)
    discs = _discs(rng, cfg, hard)
    n = H * W
    v = np.tile(dirs[0], (n, 1))
    truth = np.zeros(n, dtype=np.int32)
    v2 = v.reshape(H, W, D)
    t2 = truth.reshape(H, W)
    for k, (cy, cx, R) in enumerate(discs, start=1):
        y0, y1 = max(0, int(cy - R - 6)), min(H, int(cy + R + 7))
        x0, x1 = max(0, int(cx - R - 6)), min(W, int(cx + R + 7))
        yy, xx = np.mgrid[y0:y1, x0:x1]
        dist = np.sqrt((yy + 0.5 - cy) ** 2 + (xx + 0.5 - cx) ** 2)
        if hard:
            inside = dist <= R
            v2[y0:y1, x0:x1][inside] = dirs[k]
            t2[y0:y1, x0:x1][inside] = k
        else:
            a = 1.0 / (1.0 + np.exp(-(R - dist) / 0.7))
            blk = v2[y0:y1, x0:x1]
            v2[y0:y1, x0:x1] = (1.0 - a)[..., None] * blk + (4.0 * a)[..., None] * dirs[k]
            t2[y0:y1, x0:x1][a > 0.5] = k
    eps = np.clip(rng.standard_normal((n, D)), -3.0, 3.0)
    v /= np.sqrt(np.sum(v * v, axis=1, keepdims=True))
    x = v + cfg["sigma"] * eps
    x /= np.sqrt(np.sum(x * x, axis=1, keepdims=True))
    x *= rng.uniform(0.5, 2.0, size=(n, 1))
    return Frame(emb=np.ascontiguousarray(x, dtype=np.float32), truth=truth, H=H, W=W, D=D,
                 cells=cells, config=config, seed=int(seed))


def frame_pool(config: str, count: int, base_seed: int = 0) -> list[Frame]:
    return [make_frame(config, base_seed + i) for i in range(count)]


def min_instance_px(n: int) -> int:
    """SURVEY R22 proposal: 200 px at 512x512, scaled with the pixel count."""
    return max(1, int(round(200.0 * n / 262144.0)))


def make_blobs(n: int, seed: int, D: int = 18, k: int = 10, std: float = 0.01):
    """PAPER.md P:336 (Table 1 design): n points in D = 18 dimensions from k = 10 clusters
    (`blobs`), Gaussian noise of standard deviation 0.01, cluster directions orthogonal or opposite
    (signed basis vectors).  Equal-size clusters in random order.  Returns (emb float32 [n, D],
    truth int32 [n])."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 7777, int(n)]))
    dirs = _directions(rng, k, D)
    truth = rng.permutation(np.arange(n) % k).astype(np.int32)
    x = dirs[truth] + std * rng.standard_normal((n, D))
    return np.ascontiguousarray(x, dtype=np.float32), truth


def make_stack(T: int, seed: int, H: int = 512, W: int = 512, D: int = 16, cells: int = 30,
               radius=(20, 35), sigma: float = 0.02, drift_px: float = 0.5, turn_rad: float = 0.005):
    """C5 (BASELINE configs[4]): a temporal stack of T frames clustered jointly
    (tracking-style embeddings: one direction per cell track).  Cells drift by ~drift_px per frame
    and each track's embedding direction random-walks by ~turn_rad radians per frame; background and
    soft boundaries as in C2.  Returns (emb float32 [T*H*W, D], truth int32 [T*H*W]) in frame-major
    raster order."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 5555, T, H, W]))
    cfg = dict(H=H, W=W, D=D, cells=cells, radius=radius, sigma=sigma, boundary="soft", gap=0)
    dirs = _directions(rng, cells + 1, D)
    discs = _discs(rng, cfg, hard=False)
    vel = rng.normal(0.0, drift_px, size=(cells, 2))
    n = H * W
    emb = np.empty((T * n, D), dtype=np.float32)
    truth = np.empty(T * n, dtype=np.int32)
    yy, xx = np.mgrid[0:H, 0:W]
    for t in range(T):
        v = np.tile(dirs[0], (n, 1)).reshape(H, W, D)
        tr = np.zeros((H, W), dtype=np.int32)
        for k, (cy, cx, R) in enumerate(discs, start=1):
            cy_t = np.clip(cy + vel[k - 1, 0] * t, R + 1, H - R - 1)
            cx_t = np.clip(cx + vel[k - 1, 1] * t, R + 1, W - R - 1)
            y0, y1 = max(0, int(cy_t - R - 6)), min(H, int(cy_t + R + 7))
            x0, x1 = max(0, int(cx_t - R - 6)), min(W, int(cx_t + R + 7))
            dist = np.sqrt((yy[y0:y1, x0:x1] + 0.5 - cy_t) ** 2 + (xx[y0:y1, x0:x1] + 0.5 - cx_t) ** 2)
            a = 1.0 / (1.0 + np.exp(-(R - dist) / 0.7))
            blk = v[y0:y1, x0:x1]
            v[y0:y1, x0:x1] = (1.0 - a)[..., None] * blk + (4.0 * a)[..., None] * dirs[k]
            tr[y0:y1, x0:x1][a > 0.5] = k
        v = v.reshape(n, D)
        v /= np.sqrt(np.sum(v * v, axis=1, keepdims=True))
        x = v + sigma * np.clip(rng.standard_normal((n, D)), -3.0, 3.0)
        x /= np.sqrt(np.sum(x * x, axis=1, keepdims=True))
        emb[t * n:(t + 1) * n] = x
        truth[t * n:(t + 1) * n] = tr.reshape(n)
        # random-walk the track directions (small rotation towards a random orthogonal direction)
        for k in range(1, cells + 1):
            g = rng.standard_normal(D)
            g -= (g @ dirs[k]) * dirs[k]
            g /= np.sqrt(np.sum(g * g))
            dirs[k] = np.cos(turn_rad) * dirs[k] + np.sin(turn_rad) * g
    return emb, truth


# ------------------------------------------------------------------------------------------------
# The paper's simulation suite (NEXT-3): the section 4.2.1 data sets of Fig. 4 and the Appendix A
# overlap frames.  Data generation only.
# ------------------------------------------------------------------------------------------------

def make_circles(seed: int, n: int = 1500, k: int = 10, noise: float = 0.02):
    """PAPER.md P:331 (Fig. 4, row 1): n = 1,500 2-D points evenly in k = 10 clusters on two
    concentric circles; a cluster is an angular position, alternate clusters on the large (radius
    U[0.95, 1.05]) and small (U[0.475, 0.525]) circle ("variations ... 10% of the circles' radius");
    Gaussian noise of standard deviation 0.02 on both coordinates.  Returns (emb float32 [n, 2],
    truth int32 [n]) in random order."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 4201]))
    truth = rng.permutation(np.arange(n) % k).astype(np.int32)
    theta = 2.0 * np.pi * truth / k + 0.3
    big = truth % 2 == 0
    rad = np.where(big, rng.uniform(0.95, 1.05, n), rng.uniform(0.475, 0.525, n))
    x = np.stack([rad * np.cos(theta), rad * np.sin(theta)], axis=1) + noise * rng.standard_normal((n, 2))
    return np.ascontiguousarray(x, dtype=np.float32), truth


def make_polarized(seed: int, instances: int, n: int = 1500, background: int = 750, noise: float | None = None):
    """PAPER.md P:331 (Fig. 4, rows 2-3): polarized 2-D data with a background cluster of 750 of the
    1,500 points ("accounting for 50% of the total points") and `instances` = 7 or 3 further
    clusters sharing the rest evenly; radii ("intensity") U[1, 2]; Gaussian noise of standard deviation
    0.005 (seven instances) or 0.01 (three instances).  The k = instances + 1 cluster directions are
    evenly spaced angles.  Returns (emb float32 [n, 2], truth int32 [n]; 0 = background)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 4202, instances]))
    if noise is None:
        noise = 0.005 if instances == 7 else 0.01
    k = instances + 1
    sizes = [background] + [(n - background) // instances + (1 if j < (n - background) % instances else 0)
                            for j in range(instances)]
    truth = rng.permutation(np.repeat(np.arange(k), sizes)).astype(np.int32)
    theta = 2.0 * np.pi * truth / k + 0.2
    rad = rng.uniform(1.0, 2.0, n)
    x = np.stack([rad * np.cos(theta), rad * np.sin(theta)], axis=1) + noise * rng.standard_normal((n, 2))
    return np.ascontiguousarray(x, dtype=np.float32), truth


def make_overlap(spacing: float, H: int = 1000, W: int = 1000, D: int = 18, circles: int = 8, diameter: int = 250):
    """PAPER.md P:533-541 (Appendix A): a 1000 x 1000 x 18 frame with eight foreground circles of
    diameter 250 px, each with its own cosine embedding (signed basis directions, orthogonal to the
    background's), no noise; the overlap level is set by the distance `spacing` (px) between
    neighbouring circle centres, placed on a ring around the frame centre (spacing >= 250: no
    overlap).  Later circles are drawn over earlier ones.  Returns (emb float32 [H W, D], truth int32
    [H W]; 0 = background, k = circle k)."""
    R = diameter / 2.0
    ring = spacing / (2.0 * np.sin(np.pi / circles))  # chord between neighbours = spacing
    cy0, cx0 = H / 2.0, W / 2.0
    dirs = np.zeros((circles + 1, D))
    for k in range(circles + 1):
        dirs[k, k // 2] = 1.0 if k % 2 == 0 else -1.0
    yy, xx = np.mgrid[0:H, 0:W]
    truth = np.zeros((H, W), dtype=np.int32)
    for k in range(circles):
        a = 2.0 * np.pi * k / circles
        cy, cx = cy0 + ring * np.sin(a), cx0 + ring * np.cos(a)
        truth[(yy + 0.5 - cy) ** 2 + (xx + 0.5 - cx) ** 2 <= R * R] = k + 1
    truth = truth.reshape(-1)
    return np.ascontiguousarray(dirs[truth], dtype=np.float32), truth
