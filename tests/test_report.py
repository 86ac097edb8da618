"""Phase-timed harness and BenchReport schema 1 (report.py:28-194 mirror).

CPU: the report format and aggregation (same keys and arithmetic as the
reference's report.py, incl. loading a reference-written report as the
baseline). GPU: run_timed / benchmark through the fused timed entry point
and through the stage-by-stage protocol.
"""

import json

import numpy as np
import pytest

from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, blobs_2d, errors
from paper_1604_02700_b200 import report as R

REFERENCE_KEYS = {  # BenchReport fields of report.py:102-129 + "schema"
    "schema", "dataset", "n", "m", "backend", "p", "similarity", "params", "repetitions", "runs",
    "mean_seconds", "stddev_seconds", "affinity_share", "ari", "jaccard", "baseline", "speedup",
}


def _fake_runs(totals):
    return [{"phases": {p: t / 10 for p in R.PHASES}, "total": t} for t in totals]


def test_report_schema_and_aggregation(tmp_path):
    d = blobs_2d(60, components=3, noise=0.3, seed=0)
    base = {"schema": 1, "dataset": d.name, "backend": "parallel", "p": 8, "mean_seconds": 3.0}
    rep = R.summarize(d, GaussianRbf(1.0), PicParams(k=3), "gpu", KernelConfig(), 0,
                      _fake_runs([1.0, 2.0, 3.0]), labels=d.labels, baseline=base)
    doc = rep.to_dict()
    assert set(doc) == REFERENCE_KEYS and doc["schema"] == R.SCHEMA_VERSION == 1
    assert doc["mean_seconds"] == 2.0
    assert doc["stddev_seconds"] == pytest.approx(np.std([1.0, 2.0, 3.0]))
    assert doc["affinity_share"] == pytest.approx(0.1)
    assert doc["ari"] == 1.0 and doc["jaccard"] == 1.0
    assert doc["speedup"] == 1.5 and doc["baseline"] == f"{d.name}/parallel/p=8"
    assert doc["params"] == {"k": 3, "epsilon": 1e-5 / 60, "max_iterations": 50, "seed": 0}
    assert doc["similarity"] == {"kind": "rbf", "sigma": 1.0}
    path = tmp_path / "r.json"
    rep.write(path)
    assert R.load_report(path) == json.loads(path.read_text())


def test_load_report_rejects_other_schema(tmp_path):
    path = tmp_path / "r.json"
    path.write_text(json.dumps({"schema": 2}))
    with pytest.raises(errors.InvalidSpec):
        R.load_report(path)


def test_run_timed_rejects_cpu_backends():
    d = blobs_2d(30, components=2, noise=0.3, seed=0)
    for backend in ("serial", "parallel"):
        with pytest.raises(errors.InvalidSpec):
            R.run_timed(d, GaussianRbf(1.0), PicParams(k=2), backend=backend)
    with pytest.raises(errors.InvalidSpec):
        R.benchmark(d, GaussianRbf(1.0), PicParams(k=2), repetitions=0)


@pytest.mark.gpu
@pytest.mark.parametrize("backend", R.BACKENDS)
def test_run_timed_gpu_matches_reference_labels(golden, backend):
    z = golden("config1")
    d = DataSet(z["X"], z["truth"], name="blobs")
    run = R.run_timed(d, GaussianRbf(1.0), PicParams(k=3), backend=backend, seed=0)
    assert np.array_equal(run.labels, z["labels"])
    assert run.trace.iterations_run == int(z["iterations"])
    assert set(run.phases) == set(R.PHASES)
    assert all(t >= 0.0 for t in run.phases.values())
    assert sum(run.phases.values()) <= run.total
    if backend == "gpu":
        assert run.phases["normalize"] == 0.0  # folded into the GEMV


@pytest.mark.gpu
def test_benchmark_report_gpu(golden):
    z = golden("config1")
    d = DataSet(z["X"], z["truth"], name="blobs")
    rep, last = R.benchmark(d, GaussianRbf(1.0), PicParams(k=3), repetitions=3)
    doc = rep.to_dict()
    assert set(doc) == REFERENCE_KEYS and len(doc["runs"]) == 3
    assert doc["ari"] == 1.0
    assert 0.0 < doc["affinity_share"] < 1.0
