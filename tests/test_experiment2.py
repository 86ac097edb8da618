"""Experiment II (cli.py:230-256) on the batched small-n engine.

CPU: the sweep's host logic — subsample order/seeds and the ARI/Jaccard
statistics — equals the reference's rows when fed the reference's labels
(a test double stands in for the device batch). GPU: the batched fp64
engine reproduces every reference run (labels, embedding, iterations) and
the rows exactly; its error behaviour matches the single-problem path.
"""

import json

import numpy as np
import pytest

from paper_1604_02700_b200 import Cosine, DataSet, GaussianRbf, PicParams, errors
from paper_1604_02700_b200 import experiment as E
from paper_1604_02700_b200.datasets import gaussian_blobs, generate

from conftest import GOLDEN


def _cases():
    return json.loads((GOLDEN / "experiment2.json").read_text())


def test_default_fractions_match_reference_cli():
    assert E.DEFAULT_FRACTIONS == [i * 0.0001 for i in range(1, 10)] + [i * 0.001 for i in range(1, 10)]
    assert len(E.DEFAULT_FRACTIONS) == 18


def test_rows_from_reference_labels(monkeypatch):
    from paper_1604_02700_b200 import gpu

    for case in _cases():
        d = generate(case["kind"], 45000, 0.05, 0)
        runs = case["runs"]

        def fake_batch(datasets, kind, params, seeds, config=None, runs=runs):
            assert [s.n for s in datasets] == [r["n"] for r in runs]
            assert list(seeds) == [r["seed"] for r in runs]
            return [(np.asarray(r["labels"]), None, None) for r in runs]

        monkeypatch.setattr(gpu, "cluster_batch", fake_batch)
        rows = E.run_experiment2(d, Cosine(), PicParams(k=case["k"]), case["fractions"],
                                 case["reps"], seed=0)
        assert rows == case["rows"]


@pytest.mark.gpu
def test_batch_reproduces_reference_runs():
    from paper_1604_02700_b200 import gpu

    for case in _cases():
        d = generate(case["kind"], 45000, 0.05, 0)
        subs = E.subsamples(d, case["fractions"], case["reps"], 0)
        out = gpu.cluster_batch([s for _, _, s in subs], Cosine(), PicParams(k=case["k"]),
                                [rs for _, rs, _ in subs])
        for run, (labels, v, trace) in zip(case["runs"], out):
            assert np.array_equal(labels, run["labels"]), (case["kind"], run["fraction"])
            ref_v = np.asarray(run["v"])
            assert np.abs(v - ref_v).sum() <= 1e-10 * np.abs(ref_v).sum()
            assert trace.iterations_run == run["iterations"]
            assert trace.converged == run["converged"]


@pytest.mark.gpu
def test_experiment2_rows_on_gpu():
    for case in _cases():
        d = generate(case["kind"], 45000, 0.05, 0)
        rows = E.run_experiment2(d, Cosine(), PicParams(k=case["k"]), case["fractions"],
                                 case["reps"], seed=0)
        assert rows == case["rows"]


@pytest.mark.gpu
def test_batch_matches_single_problem_path(golden):
    from paper_1604_02700_b200 import gpu
    from paper_1604_02700_b200 import cluster

    z = golden("config1")
    d1 = DataSet(z["X"], z["truth"])
    d2 = gaussian_blobs(3000, 16, 4, seed=5)
    d3 = gaussian_blobs(700, 16, 4, seed=6)
    out = gpu.cluster_batch([d2, d3], GaussianRbf(2.0), PicParams(k=4), [1, 2])
    for d, s, (labels, v, trace) in zip((d2, d3), (1, 2), out):
        l_ref, v_ref, t_ref = cluster(d, GaussianRbf(2.0), PicParams(k=4), seed=s)
        assert np.array_equal(labels, l_ref)
        assert np.abs(v - v_ref).sum() <= 1e-4 * np.abs(v_ref).sum()
        assert abs(trace.iterations_run - t_ref.iterations_run) <= 2
    # config 1 through the batch equals the reference fixture
    (labels, v, trace), = gpu.cluster_batch([d1], GaussianRbf(1.0), PicParams(k=3), [0])
    assert np.array_equal(labels, z["labels"])
    assert np.abs(v - z["v"]).max() <= 1e-12 * np.abs(z["v"]).max()
    assert trace.iterations_run == int(z["iterations"])
    assert np.allclose(trace.delta_history, z["deltas"], rtol=1e-6, atol=0)


@pytest.mark.gpu
def test_batch_errors_match_reference():
    from paper_1604_02700_b200 import gpu

    e = json.loads((GOLDEN / "errors.json").read_text())
    ok = generate("blobs", 30, 0.3, 0)
    zd = DataSet(np.array(e["zero_degree"]["points"]))
    with pytest.raises(errors.ZeroDegree) as info:
        gpu.cluster_batch([ok, DataSet(np.pad(zd.points, ((0, 0), (0, 1))))], GaussianRbf(1.0),
                          PicParams(k=2), [0, 0])
    assert info.value.index == e["zero_degree"]["index"]
    bad = np.ones((5, 2))
    bad[3, 1] = np.nan
    with pytest.raises(errors.NonFiniteEntry) as info:
        gpu.cluster_batch([ok, DataSet(bad)], GaussianRbf(1.0), PicParams(k=2), [0, 0])
    assert (info.value.row, info.value.col) == (3, 1)
    zv = DataSet(np.array(e["zero_vector"]["points"]))
    with pytest.raises(errors.ZeroVector) as info:
        gpu.cluster_batch([ok, zv], Cosine(), PicParams(k=2), [0, 0])
    assert info.value.index == e["zero_vector"]["index"]
    with pytest.raises(errors.KTooLarge):
        gpu.cluster_batch([ok, DataSet(np.ones((2, 2)))], GaussianRbf(1.0), PicParams(k=3), [0, 0])
