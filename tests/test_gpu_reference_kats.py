"""The reference's end-to-end known-answer tests on the device engine.

Mirrors test_serial.py:124-159 (identical points collapse under the cosine
kind, the six-point block toy, power-of-two scale invariance through the
pipeline) and test_parallel.py:213-223 (chunk sizes do not change any
value) with the same inputs and the same exact assertions.
"""

import numpy as np
import pytest

from paper_1604_02700_b200 import (Cosine, DataSet, GaussianRbf, KernelConfig, KMeansParams,
                                   PicParams)

pytestmark = pytest.mark.gpu


def _gpu():
    from paper_1604_02700_b200 import gpu

    return gpu


def random_points(rng, n, d=2):
    # the reference helper's distribution (tests/oracles.py:144-146):
    # positive-quadrant points, safe for the cosine kind
    return rng.uniform(0.1, 4.0, size=(n, d))


@pytest.mark.parametrize("storage", ["packed", "dense", "none"])
def test_identical_points_collapse(storage):
    """test_serial.py:124-127: eight copies of one point, cosine kind."""
    d = DataSet(np.tile([1.0, 2.0], (8, 1)))
    cfg = KernelConfig(storage=storage, affinity_impl="simt" if storage == "dense" else "tc")
    labels, v, _ = _gpu().cluster(d, Cosine(), PicParams(k=2), cfg, seed=0)
    assert len(set(labels.tolist())) == 1
    assert np.all(v == v[0])


def test_six_point_block_toy():
    """test_serial.py:129-144: two cliques, degrees 2,2,2 and 1,1,1; the
    degree vector is an exact eigenvector, so two flat levels."""
    gpu = _gpu()
    a = np.zeros((6, 6))
    a[:3, :3] = 1.0 - np.eye(3)
    a[3:, 3:] = 0.5 * (1.0 - np.eye(3))
    deg = gpu.degree(a)
    assert np.array_equal(deg, [2.0, 2.0, 2.0, 1.0, 1.0, 1.0])
    w = gpu.normalize(a, deg)
    v0 = gpu.initial_vector(deg, "degree")
    v, trace = gpu.power_iterate(w, PicParams(k=2), v0)
    assert trace.iterations_run >= 1
    labels = gpu.kmeans_1d(v, KMeansParams(k=2, seed=0))
    assert np.array_equal(labels, [1, 1, 1, 0, 0, 0])


def test_scale_invariance_through_pipeline():
    """test_serial.py:146-159: A and 2A give the same W, v and delta
    history, bit for bit."""
    gpu = _gpu()
    rng = np.random.default_rng(42)
    d = DataSet(random_points(rng, 30))
    a1 = gpu.build_affinity(d, GaussianRbf(0.7))
    a2 = 2.0 * a1
    deg1, deg2 = gpu.degree(a1), gpu.degree(a2)
    assert np.array_equal(deg2, 2.0 * deg1)
    w1 = gpu.normalize(a1, deg1)
    w2 = gpu.normalize(a2, deg2)
    assert np.array_equal(w1.numpy(), w2.numpy())
    params = PicParams(k=2)
    v1, t1 = gpu.power_iterate(w1, params, gpu.initial_vector(deg1, "degree"))
    v2, t2 = gpu.power_iterate(w2, params, gpu.initial_vector(deg2, "degree"))
    assert np.array_equal(v1, v2)
    assert np.array_equal(t1.delta_history, t2.delta_history)


@pytest.mark.parametrize("storage", ["packed", "dense", "none"])
def test_scaled_points_and_sigma_give_identical_runs(storage):
    """The same invariance one level up: X -> 2X with sigma -> 2 sigma scales
    every distance by 4 and 2 sigma^2 by 4 exactly, so the whole device run
    (affinity, degree, iteration, k-means) is bitwise unchanged."""
    gpu = _gpu()
    rng = np.random.default_rng(7)
    pts = np.vstack([rng.normal(0.0, 0.3, (150, 12)) + c
                     for c in rng.uniform(-4.0, 4.0, (3, 12))])
    cfg = KernelConfig(storage=storage, affinity_impl="simt" if storage == "dense" else "tc")
    params = PicParams(k=3, max_iterations=30)
    l1, v1, t1 = gpu.cluster(DataSet(pts), GaussianRbf(1.1), params, cfg, seed=3)
    l2, v2, t2 = gpu.cluster(DataSet(2.0 * pts), GaussianRbf(2.2), params, cfg, seed=3)
    assert np.array_equal(l1, l2)
    assert np.array_equal(v1, v2)
    assert np.array_equal(t1.delta_history, t2.delta_history)


def test_chunking_does_not_change_values():
    """test_parallel.py:213-223: cosine kind, p = 4, chunk rows 100 / 64 / 7."""
    gpu = _gpu()
    rng = np.random.default_rng(11)
    d = DataSet(random_points(rng, 100))
    params = PicParams(k=2)
    outs = [gpu.cluster(d, Cosine(), params,
                        KernelConfig(p=4, chunk_rows=chunk, virtual_ranks=True, storage="dense",
                                     affinity_impl="simt"), seed=3)
            for chunk in (100, 64, 7)]
    for labels, v, trace in outs[1:]:
        assert np.array_equal(labels, outs[0][0])
        assert np.array_equal(v, outs[0][1])
        assert np.array_equal(trace.delta_history, outs[0][2].delta_history)
