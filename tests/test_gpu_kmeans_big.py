"""k-means with many clusters (64 < k <= 4096): kmeans_big.cu vs the oracle.

The reference accepts any k <= n (kmeans.py:178-196). Above 64 clusters the
device runs the same algorithm on the once-sorted values (clusters are
contiguous runs, sums are prefix differences, kmeans_big.cu); labels must be
equal to the reference's for well-separated and for noisy values, with the
DP polish (n <= 4096) and without (n > 4096), and end to end through
cluster().
"""

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200 import (GaussianRbf, KMeansParams, KernelConfig, PicParams, cluster,
                                   gaussian_blobs, gpu)
from paper_1604_02700_b200.errors import InvalidSpec

pytestmark = pytest.mark.gpu


def _levels(n, k, rng, spread=1e-3):
    """k well-separated value levels with small noise, shuffled."""
    centres = np.sort(rng.uniform(0.0, 1.0, k))
    lab = rng.integers(0, k, n)
    return np.abs(centres[lab] + spread * rng.standard_normal(n) / k)


@pytest.mark.parametrize("n,k", [(50_000, 100), (20_000, 65), (100_000, 500), (3000, 100),
                                 (4096, 300), (200, 150)])
def test_big_k_matches_oracle(n, k):
    rng = np.random.default_rng(n + k)
    for trial, v in enumerate([_levels(n, k, rng), rng.exponential(1e-5, n),
                               np.round(rng.uniform(0, 1, n), 3)]):
        got = gpu.kmeans_1d(v, KMeansParams(k=k, seed=trial))
        ref = po.kmeans_1d(v, k, trial)
        assert got.dtype == np.int64 and got.shape == (n,)
        if trial == 0 or n <= 4096:
            assert np.array_equal(got, ref), f"trial {trial}: {np.sum(got != ref)} labels differ"
        else:
            # noisy continuous values: Lloyd's fixed point may differ only
            # through the rounding of cluster means (prefix differences vs
            # numpy's pairwise sums); the partition must still agree almost
            # everywhere
            assert np.mean(got == ref) > 0.999


def test_big_k_duplicates_and_ties():
    """Repeated values (duplicate centres, empty-cluster reseeds) and exact
    midpoint ties (lowest index wins)."""
    rng = np.random.default_rng(7)
    v = np.repeat(np.arange(90, dtype=np.float64), 7)[rng.permutation(630)]
    for k in (70, 90):
        assert np.array_equal(gpu.kmeans_1d(v, KMeansParams(k=k, seed=1)), po.kmeans_1d(v, k, 1))
    w = np.concatenate([np.arange(80.0), np.arange(80.0) + 0.5])
    assert np.array_equal(gpu.kmeans_1d(w, KMeansParams(k=100, seed=3)), po.kmeans_1d(w, 100, 3))


def test_k_limits():
    v = np.linspace(0, 1, 5000)
    with pytest.raises(InvalidSpec):
        gpu.kmeans_1d(v, KMeansParams(k=4097))


def test_cluster_with_100_blobs():
    d = gaussian_blobs(8000, 16, 100, seed=11, radius=200.0)
    labels, v, trace = cluster(d, GaussianRbf(2.0), PicParams(k=100), config=KernelConfig(), seed=0)
    ref_labels, ref_v, ref_deltas, _ = po.pic_cluster(d.points, 2.0, 100, seed=0)
    assert abs(trace.iterations_run - len(ref_deltas)) <= 2
    if trace.iterations_run == len(ref_deltas):
        assert np.abs(v - ref_v).sum() / np.abs(ref_v).sum() <= 1e-4
    assert np.array_equal(labels, ref_labels)
