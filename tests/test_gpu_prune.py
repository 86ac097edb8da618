"""Tile pruning (csrc/prune.cu): provably-zero block pairs are never computed.

Pruning skips the tcgen05 work units of block pairs whose projection bound
puts every entry below the 2^-64 flush with two exponent units of margin,
so the run must be bit-identical to the one that computes them
(GPIC_PRUNE=0), and on well-separated, cluster-ordered data it must actually
skip most of the triangle. The near-threshold case places blob separations
around the bound (exponents ~55-80) so that pruning decisions are marginal.
"""

import ctypes as C

import numpy as np
import pytest

from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs
from paper_1604_02700_b200.datasets import config_dataset

pytestmark = pytest.mark.gpu


def _near_threshold(seed=0):
    """Blobs in d = 16 (sigma = 2) on a line, separations 15 ... 25 apart:
    cross-blob exponents log2(e) |x_i - x_j|^2 / 2 sigma^2 ~ 45 ... 120."""
    rng = np.random.default_rng(seed)
    d, per = 16, 1500
    e = rng.standard_normal(d)
    e /= np.linalg.norm(e)
    pos = np.cumsum([0.0, 15.0, 17.0, 19.0, 21.0, 23.0, 25.0])
    pts = np.vstack([p * e + rng.standard_normal((per, d)) for p in pos])
    return DataSet(pts), 2.0, len(pos)


CASES = {
    "cfg2": lambda: (config_dataset(2, 0), float(np.sqrt(32) / 2), 5),
    "near_threshold": _near_threshold,
    "blobs64_ragged": lambda: (gaussian_blobs(9001, 64, 7, seed=2), 4.0, 7),
    "blobs128": lambda: (gaussian_blobs(6000, 128, 4, seed=8, radius=60.0),
                         float(np.sqrt(128) / 2), 4),
    "shuffled": lambda: (DataSet(np.random.default_rng(1).permutation(
        gaussian_blobs(8000, 32, 6, seed=3).points)), float(np.sqrt(32) / 2), 6),
}


def _run(monkeypatch, flag, d, sigma, k, cfg, **kw):
    monkeypatch.setenv("GPIC_PRUNE", flag)
    return cluster(d, GaussianRbf(sigma), PicParams(k=k, **kw), config=cfg, seed=0)


@pytest.mark.parametrize("storage", ["packed", "packed16", "none"])
@pytest.mark.parametrize("case", list(CASES))
def test_prune_is_bitwise_neutral(monkeypatch, case, storage):
    """Packed units and the matrix-free sym pass's items (storage none)."""
    d, sigma, k = CASES[case]()
    cfg = KernelConfig(storage=storage)
    for kw in ({}, {"epsilon": 5e-324, "max_iterations": 4}):
        (la, va, ta) = _run(monkeypatch, "0", d, sigma, k, cfg, **kw)
        (lb, vb, tb) = _run(monkeypatch, "1", d, sigma, k, cfg, **kw)
        assert np.array_equal(la, lb)
        assert np.array_equal(va, vb), f"max |dv| = {np.max(np.abs(va - vb))}"
        assert ta.iterations_run == tb.iterations_run
        assert np.array_equal(ta.delta_history, tb.delta_history)


def _kept_units(d, sigma, k):
    """(units computed, units in the triangle) of one gpic_cluster run."""
    import torch

    from paper_1604_02700_b200 import _lib, gpu

    L = _lib.lib()
    dev = torch.device("cuda", 0)
    n, m = d.points.shape
    T = 50
    nbytes = gpu.workspace_bytes(n, m, k, T, 1)
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    x = torch.from_numpy(d.points).to(dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    v = torch.empty(n, dtype=torch.float64, device=dev)
    hist = torch.zeros(T, dtype=torch.float64, device=dev)
    first, u = gpu.kmeans_draws(n, k, 0)
    it, cv = C.c_int32(0), C.c_int32(0)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    rc = L.gpic_cluster(p(x), n, m, sigma, _lib.KIND_RBF, k, 1e-5 / n, T, first,
                        u.ctypes.data_as(C.c_void_p), _lib.AFFINITY_TC, 1, None, p(labels), p(v),
                        p(hist), C.byref(it), C.byref(cv), p(work), nbytes,
                        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    assert rc == 0
    offs = (C.c_int64 * 8)()
    assert L.gpic_cluster_workspace_layout(n, m, k, T, 1, offs) == 0
    kept = int(work[offs[6]: offs[6] + 8].view(torch.int64).item())
    return kept, int(offs[7])


def test_prune_skips_most_of_config3():
    kept, total = _kept_units(config_dataset(3, 0), 4.0, 10)
    print(f"config 3: {kept} of {total} units computed")
    assert 0 < kept < 0.3 * total


def test_prune_keeps_everything_when_nothing_is_provable():
    d, sigma, k = CASES["shuffled"]()
    kept, total = _kept_units(d, sigma, k)
    assert kept == total
