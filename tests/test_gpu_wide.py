"""Feature dimensions beyond the tcgen05 engine's resident K.

The reference accepts any d (affinity.py:96-101 loops over features). The
tcgen05 engine keeps the row operands in shared memory: d <= 192 for the
storing modes (d <= 256 matrix-free). The C-ABI routes wider data to the
SIMT engine with dense rows (capi.cu
effective_engine) for gpic_cluster, its workspace query, the stage-wise
affinity calls and the sharded runner; results must still match the oracle.
Tolerances as tests/test_gpu_parity.py (labels equal, v within 1e-4
relative L1 at a forced equal iteration count).
"""

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs

pytestmark = pytest.mark.gpu

TINY_EPS = 5e-324


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


@pytest.mark.parametrize("d", [192, 200, 256, 300, 700])
@pytest.mark.parametrize("storage", ["packed", "dense", "packed16"])
def test_wide_features_match_oracle(d, storage):
    g = gaussian_blobs(1500, d, 4, seed=3)
    sigma = np.sqrt(d) / 2
    params = PicParams(k=4, epsilon=TINY_EPS, max_iterations=7)
    labels, v, trace = cluster(g, GaussianRbf(sigma), params, config=KernelConfig(storage=storage))
    ref_labels, ref_v, _, _ = po.pic_cluster(g.points, sigma, 4, epsilon=TINY_EPS, max_iterations=7)
    assert trace.iterations_run == 7
    assert np.array_equal(labels, ref_labels)
    assert rel_l1(v, ref_v) <= 1e-4


def test_wide_features_stagewise_and_sharded():
    from paper_1604_02700_b200 import gpu

    g = gaussian_blobs(1200, 320, 3, seed=4)
    sigma = np.sqrt(320) / 2
    a = gpu.k_affinity(g, GaussianRbf(sigma), KernelConfig())  # tc requested, SIMT runs
    full = a.numpy()
    ref = po.affinity(g.points, sigma)
    assert np.abs(full - ref).max() <= 1e-4 * ref.max()
    params = PicParams(k=3, epsilon=TINY_EPS, max_iterations=6)
    one, v1, _ = cluster(g, GaussianRbf(sigma), params)
    two, v2, _ = cluster(g, GaussianRbf(sigma), params, config=KernelConfig(p=2, virtual_ranks=True))
    assert np.array_equal(one, two)
    assert rel_l1(v2, v1) <= 1e-5
