"""Phase-timed runs and the benchmark report format on the GPU backend.

Mirrors `picluster/report.py`: the same SCHEMA_VERSION,
PHASES, TimedRun, BenchReport (to_dict / write), load_report and benchmark
(report.py:28-194), so a report written here loads next to one written by
the reference and `benchmark(..., baseline=<reference report dict>)` fills
`speedup` = reference mean / GPU mean directly.

Timing. `total` is the host wall clock (perf_counter) around the whole call
— H2D of X, the pipeline, D2H of labels / v / deltas — like the reference's
total (report.py:59,97). The per-phase seconds are device time:

* backend "gpu": one fused `gpic_cluster_timed` call, CUDA events recorded
  on the launching stream at the phase boundaries (no host sync inside);
  "normalize" is 0 because W = D^-1 A is never formed (the GEMV applies
  1/d), "rowsum" is the degree combine of the fused epilogue partials.
* backend "gpu-stages": the reference's stage-by-stage protocol
  (k_affinity, k_rowsum, k_normalize, initial_embedding + iterate,
  kmeans_1d; report.py:80-95) on dense row storage, each stage bracketed by
  device synchronisation — the shape of the reference's "parallel" branch.

The reference's "serial" / "parallel" CPU backends are not provided (no
CPU fallback); pass their written report as ``baseline``.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .data import DataSet, check_labels, check_shape
from .errors import InvalidSpec, KTooLarge
from .params import Cosine, KernelConfig, KMeansParams, PicParams, PicTrace
from .validation import adjusted_rand_index, contingency, jaccard_index

SCHEMA_VERSION = 1
PHASES = ("affinity", "rowsum", "normalize", "iterate", "kmeans")
BACKENDS = ("gpu", "gpu-stages")


@dataclass
class TimedRun:
    labels: np.ndarray
    embedding: np.ndarray
    trace: PicTrace
    phases: dict[str, float]
    total: float


def similarity_to_dict(kind) -> dict:
    if isinstance(kind, Cosine):
        return {"kind": "cosine"}
    return {"kind": "rbf", "sigma": kind.sigma}


def _sync():
    import torch

    torch.cuda.synchronize()


def _run_stages(d, kind, params, config, seed):
    from . import gpu

    clock = time.perf_counter
    phases = {}
    t = clock()
    a = gpu.k_affinity(d, kind, config)
    _sync()
    phases["affinity"] = clock() - t
    t = clock()
    deg = gpu.k_rowsum(a, config)
    _sync()
    phases["rowsum"] = clock() - t
    t = clock()
    w = gpu.k_normalize(a, deg, config)
    _sync()
    phases["normalize"] = clock() - t
    t = clock()
    v = gpu.initial_embedding(deg, params, config)
    v, trace = gpu.iterate(w, v, params, config)
    _sync()
    phases["iterate"] = clock() - t
    del a, w
    t = clock()
    labels = gpu.kmeans_1d(v, KMeansParams(k=params.k, seed=seed), config)
    labels = labels.cpu().numpy()
    phases["kmeans"] = clock() - t
    return labels, v.cpu().numpy(), trace, phases


def run_timed(d: DataSet, kind, params: PicParams, backend: str = "gpu",
              config: KernelConfig | None = None, seed: int = 0) -> TimedRun:
    """Run one clustering pass, timing each pipeline phase (report.py:47-99)."""
    from . import gpu

    config = config or KernelConfig()
    if backend not in BACKENDS:
        raise InvalidSpec(f"unknown backend {backend!r}; phase timing runs on {BACKENDS}")
    if config.p > 1:
        raise InvalidSpec("phase timing runs on one device (p=1); time sharded runs end to end")
    gpu._check_kind(kind)
    check_shape(d)
    check_labels(d)
    if params.k > d.n:
        raise KTooLarge(params.k, d.n)
    fused = backend == "gpu"
    _sync()
    start = time.perf_counter()
    if fused:
        labels, v, trace, phases = gpu.cluster_fused(d, kind, params, config, seed, timed=True)
    else:
        labels, v, trace, phases = _run_stages(d, kind, params, config, seed)
    total = time.perf_counter() - start
    return TimedRun(labels, v, trace, phases, total)


# The report record: field names and meaning are schema 1 of the reference
# (report.py:102-129), so reports written here and there load side by side.
REPORT_FIELDS = ("dataset", "n", "m", "backend", "p", "similarity", "params", "repetitions",
                 "runs", "mean_seconds", "stddev_seconds", "affinity_share", "ari", "jaccard",
                 "baseline", "speedup")


@dataclass
class BenchReport:
    """One configuration timed `repetitions` times (schema 1 fields)."""

    dataset: str
    n: int
    m: int
    backend: str
    p: int
    similarity: dict
    params: dict
    repetitions: int
    runs: list[dict] = field(default_factory=list)
    mean_seconds: float = 0.0
    stddev_seconds: float = 0.0
    affinity_share: float = 0.0
    ari: float | None = None
    jaccard: float | None = None
    baseline: str | None = None
    speedup: float | None = None

    def to_dict(self) -> dict:
        doc = {"schema": SCHEMA_VERSION}
        doc.update((name, getattr(self, name)) for name in REPORT_FIELDS)
        return doc

    def write(self, path: str | Path) -> None:
        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n", encoding="utf-8")


def load_report(path: str | Path) -> dict:
    """A schema-1 report document (ours or the reference's)."""
    doc = json.loads(Path(path).read_text(encoding="utf-8"))
    version = doc.get("schema")
    if version != SCHEMA_VERSION:
        raise InvalidSpec(f"unsupported report schema {version!r}")
    return doc


def _baseline_tag(doc: dict) -> str:
    return "/".join((str(doc["dataset"]), str(doc["backend"]), f"p={doc['p']}"))


def summarize(d: DataSet, kind, params: PicParams, backend: str, config: KernelConfig,
              seed: int, runs: list[dict], labels=None, baseline: dict | None = None
              ) -> BenchReport:
    """Fold already-timed runs into a BenchReport: population mean / stddev
    of the totals, the affinity phase's share of all the time, pair-counting
    indices against the data's labels, speedup against a baseline report."""
    totals = np.array([r["total"] for r in runs], dtype=np.float64)
    affinity = np.array([r["phases"]["affinity"] for r in runs], dtype=np.float64)
    mean = float(totals.mean())
    report = BenchReport(
        dataset=d.name, n=d.n, m=d.m, backend=backend, p=config.p,
        similarity=similarity_to_dict(kind),
        params=dict(k=params.k, epsilon=params.resolved_epsilon(d.n),
                    max_iterations=params.max_iterations, seed=seed),
        repetitions=len(runs), runs=runs, mean_seconds=mean,
        stddev_seconds=float(totals.std()),
        affinity_share=float(affinity.sum() / totals.sum()),
    )
    if labels is not None and d.labels is not None:
        table = contingency(d.labels, labels)
        report.ari, report.jaccard = adjusted_rand_index(table), jaccard_index(table)
    if baseline is not None:
        report.baseline = _baseline_tag(baseline)
        report.speedup = baseline["mean_seconds"] / mean
    return report


def benchmark(d: DataSet, kind, params: PicParams, backend: str = "gpu",
              config: KernelConfig | None = None, seed: int = 0, repetitions: int = 1,
              baseline: dict | None = None) -> tuple[BenchReport, TimedRun]:
    """Run ``repetitions`` timed passes and aggregate them (report.py:140-194)."""
    if repetitions < 1:
        raise InvalidSpec("repetitions must be at least 1")
    config = config or KernelConfig()
    runs = []
    last: TimedRun | None = None
    for _ in range(repetitions):
        last = run_timed(d, kind, params, backend, config, seed)
        runs.append({"phases": dict(last.phases), "total": last.total})
    report = summarize(d, kind, params, backend, config, seed, runs,
                       labels=last.labels, baseline=baseline)
    return report, last
