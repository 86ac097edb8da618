"""Synthetic Gaussian-blob inputs for the benchmark configs.

* `blobs_2d` reproduces the reference's ``generate(GeneratorSpec("blobs", ...))``
  (`picluster/datasets.py:74-76,117-125,147-171`) bit for bit, so config 1
  runs on exactly the reference's points.
* `gaussian_blobs` is the d-dimensional generator of SURVEY.md App. B used
  for configs 2-5 (the reference only emits 2-D data).
* `two_moons` / `three_circles` reproduce the reference's generators of the
  same names (`datasets.py:79-98`), the inputs of the paper's Table 2
  protocol (cosine similarity); `cassine` / `shapes` /
  `smiley` (`datasets.py:101-139`) with `blobs_2d` are the Experiment-II
  datasets and `subsample_balanced` its subsampler
  (`datasets.py:174-204`); `generate(kind, ...)` dispatches like the
  reference's `generate(GeneratorSpec(...))`.

Both are deterministic for a fixed seed (numpy PCG64).
"""

from __future__ import annotations

import math

import numpy as np

from .data import DataSet
from .errors import InvalidSpec


def _even_split(n: int, c: int) -> list[int]:
    q, r = divmod(n, c)
    return [q + 1 if i < r else q for i in range(c)]


def blobs_2d(n: int, components: int = 3, noise: float = 0.3, seed: int = 0) -> DataSet:
    """Blobs on a radius-5 circle, offset (8, 8), isotropic noise."""
    if components < 1 or n < components or noise < 0:
        raise InvalidSpec("blobs needs components >= 1, n >= components, noise >= 0")
    rng = np.random.default_rng(seed)
    sizes = _even_split(n, components)
    parts = []
    for i, cnt in enumerate(sizes):
        t = 2.0 * np.pi * i / components
        parts.append(np.tile([5.0 * np.cos(t), 5.0 * np.sin(t)], (cnt, 1)))
    pts = np.vstack(parts)
    if noise > 0:
        pts = pts + noise * rng.standard_normal(pts.shape)
    pts = pts + np.asarray((8.0, 8.0))
    lab = np.concatenate([np.full(c, i, dtype=np.int64) for i, c in enumerate(sizes)])
    return DataSet(pts, lab, name="blobs")


def _finish(groups, sizes, offset, noise, rng, name):
    # stack the noiseless geometry, jitter it, then translate (datasets.py:155-171)
    pts = np.vstack(groups)
    if noise > 0:
        pts = pts + noise * rng.standard_normal(pts.shape)
    pts = pts + np.asarray(offset)
    lab = np.concatenate([np.full(c, i, dtype=np.int64) for i, c in enumerate(sizes)])
    return DataSet(pts, lab, name=name)


def _ring(count: int, lo: float, hi: float, r: float, cx: float, cy: float, closed: bool):
    t = np.linspace(lo, hi, count, endpoint=not closed)
    return np.column_stack([cx + r * np.cos(t), cy + r * np.sin(t)])


def two_moons(n: int, noise: float = 0.05, seed: int = 0) -> DataSet:
    """Interleaved unit half circles, offset (3, 2) (datasets.py:79-84)."""
    if n < 2 or noise < 0:
        raise InvalidSpec("two-moons needs n >= 2 and noise >= 0")
    rng = np.random.default_rng(seed)
    sizes = _even_split(n, 2)
    top = _ring(sizes[0], 0.0, np.pi, 1.0, 0.0, 0.0, closed=False)
    bottom = _ring(sizes[1], 0.0, np.pi, 1.0, 1.0, 0.5, closed=False)
    bottom[:, 1] = 1.0 - bottom[:, 1]
    return _finish([top, bottom], sizes, (3.0, 2.0), noise, rng, "two-moons")


def three_circles(n: int, noise: float = 0.05, seed: int = 0) -> DataSet:
    """Concentric circles of radii 1, 2, 3, offset (5, 4) (datasets.py:87-98)."""
    if n < 3 or noise < 0:
        raise InvalidSpec("three-circles needs n >= 3 and noise >= 0")
    rng = np.random.default_rng(seed)
    sizes = _even_split(n, 3)
    rings = [_ring(c, 0.0, 2.0 * np.pi, float(i + 1), 0.0, 0.0, closed=True)
             for i, c in enumerate(sizes)]
    return _finish(rings, sizes, (5.0, 4.0), noise, rng, "three-circles")


def cassine(n: int, noise: float = 0.05, seed: int = 0) -> DataSet:
    """Two interlocking radius-2 arcs, offset (6, 5) (datasets.py:101-108)."""
    if n < 2 or noise < 0:
        raise InvalidSpec("cassine needs n >= 2 and noise >= 0")
    rng = np.random.default_rng(seed)
    sizes = _even_split(n, 2)
    a = np.deg2rad(115.0)
    left = _ring(sizes[0], -a, a, 2.0, 0.0, 0.0, closed=False)
    right = _ring(sizes[1], np.deg2rad(65.0), np.deg2rad(295.0), 2.0, 2.4, 0.0, closed=False)
    return _finish([left, right], sizes, (6.0, 5.0), noise, rng, "cassine")


def shapes(n: int, noise: float = 0.05, seed: int = 0) -> DataSet:
    """Blob, square, ring and sine wave on a square's corners, offset (7, 7)
    (datasets.py:122-130). The blob and square draw from the same PCG64
    stream as the noise, in that order."""
    if n < 4 or noise < 0:
        raise InvalidSpec("shapes needs n >= 4 and noise >= 0")
    rng = np.random.default_rng(seed)
    c = _even_split(n, 4)
    blob = 0.4 * rng.standard_normal((c[0], 2)) + [-2.5, -2.5]
    square = rng.uniform(-0.8, 0.8, size=(c[1], 2)) + [2.5, -2.5]
    ring = _ring(c[2], 0.0, 2.0 * np.pi, 1.0, 0.0, 0.0, closed=True) + [-2.5, 2.5]
    t = np.linspace(-1.0, 1.0, c[3])
    wave = np.column_stack([t, 0.5 * np.sin(3.0 * t)]) + [2.5, 2.5]
    return _finish([blob, square, ring, wave], c, (7.0, 7.0), noise, rng, "shapes")


def smiley(n: int, noise: float = 0.05, seed: int = 0) -> DataSet:
    """Two eyes, a nose and a mouth arc, offset (6, 6) (datasets.py:133-139)."""
    if n < 4 or noise < 0:
        raise InvalidSpec("smiley needs n >= 4 and noise >= 0")
    rng = np.random.default_rng(seed)
    c = _even_split(n, 4)
    eye_l = 0.25 * rng.standard_normal((c[0], 2)) + [-1.2, 1.0]
    eye_r = 0.25 * rng.standard_normal((c[1], 2)) + [1.2, 1.0]
    nose = rng.standard_normal((c[2], 2)) * [0.12, 0.35] + [0.0, -0.2]
    mouth = _ring(c[3], np.deg2rad(200.0), np.deg2rad(340.0), 2.0, 0.0, 0.6, closed=False)
    return _finish([eye_l, eye_r, nose, mouth], c, (6.0, 6.0), noise, rng, "smiley")


def generate(kind: str, n: int, noise: float = 0.0, seed: int = 0,
             components: int = 3) -> DataSet:
    """The reference's `generate(GeneratorSpec(kind, ...))` (datasets.py:147-171)."""
    if kind == "blobs":
        return blobs_2d(n, components=components, noise=noise, seed=seed)
    makers = {"two-moons": two_moons, "three-circles": three_circles, "cassine": cassine,
              "shapes": shapes, "smiley": smiley}
    if kind not in makers:
        raise InvalidSpec(f"unknown generator kind {kind!r}; choose from "
                          f"{tuple(makers) + ('blobs',)}")
    return makers[kind](n, noise, seed)


def subsample_balanced(d: DataSet, fraction: float, seed: int = 0) -> DataSet:
    """Equal-size class sample without replacement (datasets.py:174-204).

    Per-class count = floor(fraction * n / classes + 0.5), clamped to
    [1, smallest class]; one PCG64 stream draws the classes in order.
    """
    from .errors import FractionTooSmall, MissingLabels

    if not (0.0 < fraction <= 1.0):
        raise FractionTooSmall(fraction)
    if d.labels is None:
        raise MissingLabels()
    rng = np.random.default_rng(seed)
    members = [np.flatnonzero(d.labels == c) for c in range(int(d.labels.max()) + 1)]
    per = int(np.floor(fraction * d.n / len(members) + 0.5))
    per = max(1, min(per, min(m.size for m in members)))
    sel = np.concatenate([rng.choice(m, size=per, replace=False) for m in members])
    return DataSet(d.points[sel].copy(), d.labels[sel].copy(), name=f"{d.name}#f={fraction}")


def graded_sizes(n: int, k: int) -> np.ndarray:
    w = np.linspace(1.0, 2.0, k)
    counts = np.floor(n * w / w.sum()).astype(np.int64)
    counts[-1] += n - counts.sum()
    return counts


def gaussian_blobs(n: int, d: int, k: int, seed: int = 0, noise: float = 1.0,
                   radius: float = 40.0, offset: float = 8.0,
                   sizes: str = "graded") -> DataSet:
    """k centres on a radius-`radius` sphere in R^d, unit noise."""
    if k < 1 or n < k or d < 1:
        raise InvalidSpec("gaussian_blobs needs k >= 1, n >= k, d >= 1")
    rng = np.random.default_rng(seed)
    if sizes == "graded":
        counts = graded_sizes(n, k)
    elif sizes == "balanced":
        counts = np.asarray(_even_split(n, k), dtype=np.int64)
    else:
        raise InvalidSpec(f"sizes must be 'graded' or 'balanced', got {sizes!r}")
    centers = rng.standard_normal((k, d))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    centers *= radius
    pts = np.vstack([centers[i] + noise * rng.standard_normal((int(counts[i]), d))
                     for i in range(k)]) + offset
    lab = np.repeat(np.arange(k, dtype=np.int64), counts)
    return DataSet(pts, lab, name=f"gblobs-n{n}-d{d}-k{k}-s{seed}")


def default_sigma(d: int) -> float:
    """sigma = sqrt(d) / 2 for the App. B configs."""
    return math.sqrt(d) / 2.0


# BASELINE.json configs: (n, d, k, sigma, generator)
CONFIGS = {
    1: dict(n=1000, d=2, k=3, sigma=1.0),
    2: dict(n=20_000, d=32, k=5, sigma=default_sigma(32)),
    3: dict(n=100_000, d=64, k=10, sigma=default_sigma(64)),
    4: dict(n=200_000, d=128, k=20, sigma=default_sigma(128)),
    5: dict(n=1_000_000, d=64, k=50, sigma=default_sigma(64)),
}


def config_dataset(cfg: int, seed: int = 0) -> DataSet:
    c = CONFIGS[cfg]
    if cfg == 1:
        return blobs_2d(c["n"], components=c["k"], noise=0.3, seed=seed)
    return gaussian_blobs(c["n"], c["d"], c["k"], seed=seed)
