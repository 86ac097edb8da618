"""Synthetic Gaussian-blob inputs for the benchmark configs.

* `blobs_2d` reproduces the reference's ``generate(GeneratorSpec("blobs", ...))``
  (`picluster/datasets.py:74-76,117-125,147-171`) bit for bit, so config 1
  runs on exactly the reference's points.
* `gaussian_blobs` is the d-dimensional generator of SURVEY.md App. B used
  for configs 2-5 (the reference only emits 2-D data).

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
