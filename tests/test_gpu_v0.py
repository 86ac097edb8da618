"""Start-vector choices on every path (serial.py:77-101, parallel.py:210-214).

The reference honours PicParams.v0 ("degree", "uniform" or an explicit
vector) for any worker count; so must the fused single-rank call and the
sharded path (the sharded loop used to start from d / sum(d)
regardless).
"""

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, errors

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TINY_EPS = 5e-324


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def _v0(n):
    v = np.random.default_rng(11).random(n) + 0.5
    return v / v.sum()


CONFIGS = [KernelConfig(), KernelConfig(storage="dense"), KernelConfig(storage="none"),
           KernelConfig(p=2, virtual_ranks=True), KernelConfig(p=3, virtual_ranks=True, storage="dense"),
           KernelConfig(p=2, virtual_ranks=True, storage="none")]


@pytest.mark.parametrize("cfg", CONFIGS, ids=[f"{c.storage}-p{c.p}" for c in CONFIGS])
@pytest.mark.parametrize("choice", ["uniform", "explicit"])
def test_start_vector_is_honoured(cfg, choice):
    z = np.load(GOLDEN / "config1.npz")
    x = z["X"]
    v0 = "uniform" if choice == "uniform" else _v0(x.shape[0])
    params = PicParams(k=3, v0=v0, epsilon=TINY_EPS, max_iterations=4)
    _, v, tr = cluster(DataSet(x), GaussianRbf(1.0), params, config=cfg)
    _, ref, _, _ = po.pic_cluster(x, 1.0, 3, epsilon=TINY_EPS, max_iterations=4, v0=v0)
    assert tr.iterations_run == 4
    assert rel_l1(v, ref) <= 1e-4
    # and it differs from the degree start (the choice is not ignored)
    _, vd, _, _ = po.pic_cluster(x, 1.0, 3, epsilon=TINY_EPS, max_iterations=4)
    assert rel_l1(v, vd) > 10 * rel_l1(v, ref)


@pytest.mark.parametrize("p", [1, 2])
def test_invalid_start_vector_raises(p):
    z = np.load(GOLDEN / "config1.npz")
    cfg = KernelConfig(p=p, virtual_ranks=p > 1)
    for bad in ("bogus", np.full(10, 0.1), -_v0(1000), _v0(1000) * 2):
        with pytest.raises(errors.InvalidSpec):
            cluster(DataSet(z["X"]), GaussianRbf(1.0), PicParams(k=3, v0=bad), config=cfg)
