"""Block sparsity (csrc/sparse.cu + csrc/prune.cu) changes no bit of the result.

32 x 32 boxes whose values all flush to zero are not stored and not read
(sparse.cu), and block pairs proved to hold only such values are not even
computed (prune.cu, projection bound with an exponent margin); since an exact
zero adds nothing to any fp32 / fp64 sum, labels, embedding and delta history
must equal the dense run's bit for bit (GPIC_SPARSE=0 turns both off).
"""

import numpy as np
import pytest

from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs
from paper_1604_02700_b200.datasets import config_dataset

pytestmark = pytest.mark.gpu


def _both(monkeypatch, d, sigma, k, cfg, **kw):
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("GPIC_SPARSE", flag)
        out.append(cluster(d, GaussianRbf(sigma), PicParams(k=k, **kw), config=cfg, seed=0))
    return out


def _same(a, b):
    (la, va, ta), (lb, vb, tb) = a, b
    assert np.array_equal(la, lb)
    assert np.array_equal(va, vb), f"max |dv| = {np.max(np.abs(va - vb))}"
    assert ta.iterations_run == tb.iterations_run
    assert np.array_equal(ta.delta_history, tb.delta_history)


CASES = {
    "cfg2": lambda: (config_dataset(2, 0), float(np.sqrt(32) / 2), 5),
    "blobs16": lambda: (gaussian_blobs(5000, 16, 6, seed=3), 2.0, 6),
    "shuffled": lambda: (DataSet(np.random.default_rng(1).permutation(
        gaussian_blobs(5000, 16, 6, seed=3).points)), 2.0, 6),
    "one_blob": lambda: (gaussian_blobs(3000, 16, 2, seed=4, radius=1.0), 8.0, 2),
    "d2": lambda: (gaussian_blobs(6000, 2, 4, seed=5), float(np.sqrt(2) / 2), 4),
    "ragged": lambda: (gaussian_blobs(4099, 24, 5, seed=6), float(np.sqrt(24) / 2), 5),
}


@pytest.mark.parametrize("storage", ["packed", "packed16"])
@pytest.mark.parametrize("case", list(CASES))
def test_sparse_equals_dense_bitwise(monkeypatch, case, storage):
    d, sigma, k = CASES[case]()
    _same(*_both(monkeypatch, d, sigma, k, KernelConfig(storage=storage)))
    _same(*_both(monkeypatch, d, sigma, k, KernelConfig(storage=storage),
                 epsilon=5e-324, max_iterations=4))


def test_sparse_config3_bitwise(monkeypatch):
    d = config_dataset(3, 0)
    _same(*_both(monkeypatch, d, 4.0, 10, KernelConfig()))
