"""Locality order (csrc/locality.cu): randomly ordered inputs are permuted so
that block sparsity and tile pruning apply, then v is scattered back.

PIC is permutation-equivariant and the labels are canonical (ordered by
centroid), so a shuffled input must give the shuffled labels of the ordered
run and, against the CPU reference, the same labels and v within the gate;
the reordered run must also actually prune.
"""

import numpy as np
import pytest

from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs
from paper_1604_02700_b200.datasets import config_dataset

from conftest import GOLDEN
from test_gpu_prune import _kept_units

pytestmark = pytest.mark.gpu


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def _shuffled(d, seed=0):
    perm = np.random.default_rng(seed).permutation(d.n)
    return DataSet(d.points[perm]), perm


def test_shuffled_config2_matches_cpu_reference():
    z = dict(np.load(GOLDEN / "config2.npz"))
    d = config_dataset(2, 0)
    sh, perm = _shuffled(d, 1)
    kind = GaussianRbf(float(z["sigma"]))
    labels, v, trace = cluster(sh, kind, PicParams(k=int(z["k"])), seed=0)
    assert np.array_equal(labels, z["labels"].astype(np.int64)[perm])
    assert abs(trace.iterations_run - int(z["iterations"])) <= 2
    _, v3, _ = cluster(sh, kind, PicParams(k=int(z["k"]), epsilon=5e-324, max_iterations=3), seed=0)
    assert rel_l1(v3, z["v_T3"][perm]) <= 1e-4


@pytest.mark.parametrize("storage", ["packed", "packed16", "none"])
def test_shuffled_equals_ordered_run(storage):
    d = gaussian_blobs(30000, 32, 6, seed=2)
    sh, perm = _shuffled(d, 3)
    kind, params = GaussianRbf(float(np.sqrt(32) / 2)), PicParams(k=6)
    cfg = KernelConfig(storage=storage)
    lo, vo, to = cluster(d, kind, params, config=cfg, seed=0)
    ls, vs, ts = cluster(sh, kind, params, config=cfg, seed=0)
    assert np.array_equal(ls, lo[perm])
    assert ts.iterations_run == to.iterations_run
    assert rel_l1(vs, vo[perm]) <= 1e-6


def test_forced_reorder_of_ordered_data(monkeypatch):
    d = gaussian_blobs(20000, 64, 5, seed=4)
    kind, params = GaussianRbf(4.0), PicParams(k=5)
    base = cluster(d, kind, params, seed=0)
    monkeypatch.setenv("GPIC_REORDER", "2")
    got = cluster(d, kind, params, seed=0)
    assert np.array_equal(got[0], base[0])
    assert rel_l1(got[1], base[1]) <= 1e-6


def test_reordered_run_prunes(monkeypatch):
    d = config_dataset(3, 0)
    sh, _ = _shuffled(d, 5)
    kept, total = _kept_units(sh, 4.0, 10)
    print(f"shuffled config 3: {kept} of {total} units computed")
    assert kept < 0.35 * total
    monkeypatch.setenv("GPIC_REORDER", "0")
    kept0, _ = _kept_units(sh, 4.0, 10)
    assert kept0 == total
