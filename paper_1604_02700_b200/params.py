"""Parameter records, field-compatible with the reference.

* `GaussianRbf` — `picluster/affinity.py:27-35`
* `PicParams`, `PicTrace` — `picluster/serial.py:23-60`
* `KMeansParams` — `picluster/kmeans.py:25-36`
* `KernelConfig` — `picluster/parallel.py:44-77`, extended with the GPU knobs.

Both similarity kinds of the reference run on the device: `GaussianRbf`
(`affinity.py:27-35`) and `Cosine` (`affinity.py:22-24`, SURVEY.md §8 f1:
unit rows in fp64, the same Gram engines, max(0, cos) epilogue, ZeroVector
for a zero row).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidSpec


@dataclass(frozen=True)
class GaussianRbf:
    """A_ij = exp(-|x_i - x_j|^2 / (2 sigma^2))."""

    sigma: float

    def __post_init__(self) -> None:
        if not (self.sigma > 0):
            raise InvalidSpec(f"sigma must be positive, got {self.sigma!r}")


@dataclass(frozen=True)
class Cosine:
    """A_ij = max(0, x_i.x_j / (|x_i| |x_j|)) (affinity.py:22-24, 41-53, 88-95)."""


SimilarityKind = GaussianRbf | Cosine


@dataclass(frozen=True)
class PicParams:
    """k, stop threshold, iteration cap and start vector (serial.py:23-47)."""

    k: int
    epsilon: float | None = None
    max_iterations: int = 50
    v0: str | np.ndarray = "degree"

    def __post_init__(self) -> None:
        if self.k < 2:
            raise InvalidSpec(f"k must be at least 2, got {self.k}")
        if self.epsilon is not None and not (self.epsilon > 0):
            raise InvalidSpec(f"epsilon must be positive, got {self.epsilon!r}")
        if self.max_iterations < 1:
            raise InvalidSpec("max_iterations must be at least 1")

    def resolved_epsilon(self, n: int) -> float:
        """A user epsilon is used verbatim; None means 1e-5 / n (serial.py:46-47)."""
        return float(self.epsilon) if self.epsilon is not None else 1e-5 / n


@dataclass(frozen=True)
class PicTrace:
    """iterations_run, delta_history[t] = max|v_(t+1) - v_t|, converged (serial.py:50-60)."""

    iterations_run: int
    delta_history: np.ndarray
    converged: bool


@dataclass(frozen=True)
class KMeansParams:
    k: int
    max_rounds: int = 100
    seed: int = 0
    tol: float = 1e-12

    def __post_init__(self) -> None:
        if self.k < 2:
            raise InvalidSpec(f"k must be at least 2, got {self.k}")
        if self.max_rounds < 1:
            raise InvalidSpec("max_rounds must be at least 1")


DEFAULT_MEMORY_BUDGET = 256 * 1024 * 1024

AFFINITY_IMPLS = ("tc", "simt")
STORAGES = ("packed", "dense", "none", "packed16")


@dataclass(frozen=True)
class KernelConfig:
    """Shard count and block sizing (parallel.py:44-77) plus GPU knobs.

    ``p`` is the number of contiguous row shards. On the GPU backend each
    shard is a rank: a real process/GPU under torch.distributed, or — when
    ``virtual_ranks`` is set — P shards executed back to back on one device
    with the identical exchange code path (the reference's bitwise
    p-invariance tests, test_parallel.py:194-223, become GPU-count
    invariance tests this way). ``chunk_rows`` / ``memory_budget_bytes``
    keep their reference meaning for the host port; the GPU builds whole
    row shards in one launch. ``affinity_impl`` picks the Gram engine:
    "tc" (tcgen05, 3-term fp16 split, default) or "simt" (FP32 FFMA, the
    comparator).
    ``storage`` = "packed" keeps only the upper triangle of 128x128 tiles
    of the (exactly symmetric) affinity matrix — half the HBM bytes of the
    affinity store and of every power iteration; "dense" keeps full rows
    (used by the SIMT engine and by row-sharded multi-rank runs); "none" is
    matrix-free: A is recomputed from X for every product (n^2 > HBM);
    "packed16" is "packed" with fp16 values (opt-in compressed W: half the
    bytes again, degrees from the stored values, fp32 accumulation).
    """

    p: int = 1
    chunk_rows: int | None = None
    memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET
    affinity_impl: str = "tc"
    virtual_ranks: bool = False
    device: int | None = None
    storage: str = "packed"

    def __post_init__(self) -> None:
        if self.p < 1:
            raise InvalidSpec(f"worker count must be at least 1, got {self.p}")
        if self.chunk_rows is not None and self.chunk_rows < 1:
            raise InvalidSpec("chunk_rows must be at least 1")
        if self.memory_budget_bytes < 8:
            raise InvalidSpec("memory budget must be positive")
        if self.affinity_impl not in AFFINITY_IMPLS:
            raise InvalidSpec(f"affinity_impl must be one of {AFFINITY_IMPLS}")
        if self.storage not in STORAGES:
            raise InvalidSpec(f"storage must be one of {STORAGES}")

    def storage_code(self) -> int:
        """GPIC_STORAGE_*: packed symmetric tiles need a single rank (either
        engine); fp16 tiles and matrix-free ("none") need the tcgen05 engine."""
        if self.storage == "none":
            if self.affinity_impl != "tc":
                raise InvalidSpec("matrix-free storage runs on the tcgen05 engine")
            return 2
        if self.storage == "packed16":
            if self.affinity_impl != "tc" or self.p != 1:
                raise InvalidSpec("fp16 packed storage runs on the tcgen05 engine, one rank")
            return 3
        if self.storage == "packed" and self.p == 1:
            return 1
        return 0

    def resolved_chunk_rows(self, n: int) -> int:
        if self.chunk_rows is not None:
            if self.chunk_rows * n * 8 > self.memory_budget_bytes:
                raise InvalidSpec(
                    f"chunk_rows={self.chunk_rows} needs {self.chunk_rows * n * 8} bytes "
                    f"per block, over the budget of {self.memory_budget_bytes}"
                )
            return min(self.chunk_rows, n)
        return max(1, min(n, self.memory_budget_bytes // (8 * n)))


@dataclass(frozen=True)
class PartitionPlan:
    """Disjoint contiguous half-open row ranges covering [0, n) (parallel.py:80-87)."""

    ranges: tuple[tuple[int, int], ...]

    def __iter__(self):
        return iter(self.ranges)

    def __len__(self):
        return len(self.ranges)


def plan_rows(n: int, p: int) -> PartitionPlan:
    """At most p contiguous ranges of ceil(n/p) rows (parallel.py:90-98)."""
    if n < 1:
        raise InvalidSpec("cannot partition an empty row space")
    if p < 1:
        raise InvalidSpec("p must be at least 1")
    step = -(-n // p)
    return PartitionPlan(tuple((lo, min(lo + step, n)) for lo in range(0, n, step)))
