"""Data-driven engine routing: large spread against sigma.

The tensor engine's Gram form |x_i|^2 + |x_j|^2 - 2 x_i.x_j carries an error
of ~2^-24 R^2 / (2 sigma^2) per entry (R^2 = max squared distance to the
mean). gpic_cluster reads R^2 from the prepare pass and runs the SIMT
difference form when that exceeds a tenth of the 1e-4 gate (capi.cu
effective_engine); these cases (R / sigma ~ 100) would break the gate on the
tensor engine.
"""

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200 import (
    DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs)
from paper_1604_02700_b200.datasets import config_dataset

pytestmark = pytest.mark.gpu

TINY_EPS = 5e-324


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def _wide(d):
    g = gaussian_blobs(3000, d, 3, seed=21, noise=0.25, radius=100.0, offset=8.0)
    return g.points, 1.0


@pytest.mark.parametrize("storage", ["packed", "dense"])
@pytest.mark.parametrize("d", [16, 64])
def test_large_spread_holds_the_gate(d, storage):
    x, sigma = _wide(d)
    xc = x - x.mean(0)
    assert np.sqrt((xc * xc).sum(1).max()) / sigma > 70  # R^2 / 2 sigma^2 > 2500: SIMT
    ref_labels, _, ref_deltas, _ = po.pic_cluster(x, sigma, 3, seed=0)
    labels, v, trace = cluster(DataSet(x), GaussianRbf(sigma), PicParams(k=3),
                               config=KernelConfig(storage=storage), seed=0)
    assert np.array_equal(labels, ref_labels)
    assert abs(trace.iterations_run - len(ref_deltas)) <= 2
    _, v5, _ = cluster(DataSet(x), GaussianRbf(sigma), PicParams(k=3, epsilon=TINY_EPS, max_iterations=5),
                       config=KernelConfig(storage=storage))
    _, r5, _, _ = po.pic_cluster(x, sigma, 3, epsilon=TINY_EPS, max_iterations=5)
    assert rel_l1(v5, r5) <= 1e-4


def test_prepare_reports_the_spread_and_config3_stays_on_tensor_cores():
    import torch

    from paper_1604_02700_b200 import _lib, gpu

    dev = torch.device("cuda", 0)
    for x, sigma, want in ((_wide(64)[0], 1.0, "simt"),
                           (config_dataset(3, 0).points, 4.0, "tc"),
                           (config_dataset(2, 0).points, float(np.sqrt(32) / 2), "tc")):
        prep = gpu.prepare_points(DataSet(x), dev)
        xc = x - x.mean(0)
        r2 = (xc * xc).sum(1).max()
        assert abs(prep.spread2 - r2) <= 1e-5 * r2
        assert prep.engine(sigma, "tc", _lib.STORAGE_PACKED) == want
