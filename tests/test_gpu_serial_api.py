"""The serial-module entry points on the device engine.

Mirrors the reference's TestPowerIterate / TestInitialVector
(test_serial.py:31-112) against `gpu.power_iterate`,
`gpu.check_row_stochastic` (device row scan, gpic_row_stats),
`build_affinity`, `degree`, `normalize` and `initial_vector`, with the
oracle (serial.py restated) as the checker. W is streamed in fp32, so the
reference's exact-equality assertions become the fp32 tolerance of
DESIGN.md §2 (v within 1e-6 absolute at these sizes; labels exact).
"""

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200 import DataSet, GaussianRbf, PicParams, errors, gaussian_blobs

pytestmark = pytest.mark.gpu

TINY_EPS = 5e-324


def _gpu():
    from paper_1604_02700_b200 import gpu

    return gpu


def random_row_stochastic(rng, n):
    w = rng.uniform(0.1, 1.0, (n, n))
    return w / w.sum(axis=1, keepdims=True)


def test_identity_fixed_point():
    v0 = np.full(3, 1.0 / 3.0)
    v, trace = _gpu().power_iterate(np.eye(3), PicParams(k=2, epsilon=1e-8, max_iterations=50), v0)
    assert np.abs(v - v0).max() <= 1e-7
    assert trace.converged and trace.iterations_run == 2


def test_swap_fixed_point():
    w = np.array([[0.0, 1.0], [1.0, 0.0]])
    v0 = np.array([0.5, 0.5])
    v, trace = _gpu().power_iterate(w, PicParams(k=2, epsilon=1e-8, max_iterations=50), v0)
    assert np.abs(v - v0).max() <= 1e-7
    assert trace.converged and trace.iterations_run == 2


def test_block_diagonal_flat_per_block():
    rng = np.random.default_rng(2)
    w = np.zeros((6, 6))
    w[:3, :3] = random_row_stochastic(rng, 3)
    w[3:, 3:] = random_row_stochastic(rng, 3)
    v, _ = _gpu().power_iterate(w, PicParams(k=2, epsilon=TINY_EPS, max_iterations=50),
                                np.full(6, 1.0 / 6.0))
    assert np.ptp(v[:3]) <= 1e-6 and np.ptp(v[3:]) <= 1e-6


def test_l1_mass_and_nonnegativity_each_iteration():
    w = random_row_stochastic(np.random.default_rng(4), 12)
    v0 = np.full(12, 1.0 / 12.0)
    for t in range(1, 6):
        # the uniform v0 is W's right eigenvector (W 1 = 1), so both engines
        # stop once two rounding-level deltas agree; only the iterate is compared
        v, trace = _gpu().power_iterate(w, PicParams(k=2, epsilon=TINY_EPS, max_iterations=t), v0)
        assert trace.iterations_run <= t
        assert abs(np.abs(v).sum() - 1.0) <= 1e-9
        assert v.min() >= 0.0
        ref, _, _ = po.power_iteration(w, v0, TINY_EPS, t)
        assert np.abs(v - ref).max() <= 1e-7


def test_trace_contract():
    rng = np.random.default_rng(6)
    for seed in range(10):
        w = random_row_stochastic(np.random.default_rng(seed), 8)
        params = PicParams(k=2, epsilon=1e-6, max_iterations=int(rng.integers(1, 30)))
        _, trace = _gpu().power_iterate(w, params, np.full(8, 1.0 / 8.0))
        assert trace.iterations_run <= params.max_iterations
        assert len(trace.delta_history) == trace.iterations_run
        if trace.converged:
            d = trace.delta_history
            assert abs(d[-1] - d[-2]) <= params.epsilon


def test_converges_to_dominant_eigenvector():
    for seed in range(5):
        w = random_row_stochastic(np.random.default_rng(100 + seed), 32)
        v, _ = _gpu().power_iterate(w, PicParams(k=2, epsilon=TINY_EPS, max_iterations=500),
                                    np.full(32, 1.0 / 32.0))
        vals, vecs = np.linalg.eig(w)
        ref = np.abs(np.real(vecs[:, np.argmax(np.real(vals))]))
        cos = float(v @ ref / (np.linalg.norm(v) * np.linalg.norm(ref)))
        assert cos >= 1.0 - 1e-6


@pytest.mark.parametrize("bad", [
    np.ones((2, 2)),                                  # rows sum to 2
    np.array([[0.5, 0.5], [0.5, 0.5 + 2e-9]]),        # just outside 1e-9
    np.array([[1.5, -0.5], [0.0, 1.0]]),              # sums fine, range not
    np.ones((2, 3)) / 3.0,                            # not square
])
def test_rejects_non_stochastic(bad):
    with pytest.raises(errors.InvalidSpec):
        _gpu().power_iterate(bad, PicParams(k=2), np.full(bad.shape[0], 1.0 / bad.shape[0]))


def test_row_scan_matches_oracle_verdict():
    """Device scan vs the oracle's verdict on random near-stochastic matrices,
    including the worst-row index the message names."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(1, 300))
        w = random_row_stochastic(rng, n)
        if trial % 3 == 1:
            i = int(rng.integers(0, n))
            w[i, int(rng.integers(0, n))] += float(rng.choice([3e-9, -3e-9, 1e-3]))
        elif trial % 3 == 2:
            w[int(rng.integers(0, n)), 0] = float(rng.choice([np.nan, 1.5, -1e-6]))
        verdict = po.row_stochastic_violation(w)
        if verdict is None:
            out = _gpu().check_row_stochastic(w)
            assert np.array_equal(out, w, equal_nan=True)
        else:
            with pytest.raises(errors.InvalidSpec) as ei:
                _gpu().check_row_stochastic(w)
            if verdict[0] == "row":
                assert str(ei.value).startswith(f"row {verdict[1]} ")
            else:
                assert "[0, 1]" in str(ei.value)


def test_serial_names_compose_like_the_reference():
    """build_affinity -> degree -> normalize -> initial_vector -> power_iterate
    (test_serial.py:130-160 shape) against the oracle pipeline."""
    # compact blobs: the fp32-class operands put ~2^-22 |x| into each
    # coordinate, i.e. a relative A error ~ 4 |x| dx sqrt(d) / (2 sigma^2)
    # (DESIGN.md §3); at radius 4 that is far below the 1e-4 bound
    d = gaussian_blobs(300, 4, 3, seed=5, radius=4.0, offset=0.0)
    sigma = 0.8
    gpu = _gpu()
    a = gpu.build_affinity(d, GaussianRbf(sigma))
    a_ref = po.affinity(d.points, sigma)
    assert a.dtype == np.float64 and a.shape == (300, 300)
    assert np.abs(a - a_ref).max() <= 1e-4 * a_ref.max()
    assert np.all(np.diag(a) == 0.0)
    deg = gpu.degree(a)
    assert np.allclose(deg, po.degree(a_ref), rtol=1e-4)
    # a host fp64 matrix is summed in fp64, as the reference does
    assert np.allclose(gpu.degree(a_ref), po.degree(a_ref), rtol=1e-14, atol=0)
    w = gpu.normalize(a, deg)
    v0 = gpu.initial_vector(deg, "degree")
    assert np.allclose(v0, deg / deg.sum(), rtol=1e-12, atol=0)
    params = PicParams(k=3, epsilon=TINY_EPS, max_iterations=8)
    v, trace = gpu.power_iterate(w, params, v0)
    ref, _, _ = po.power_iteration(po.normalize(a_ref, po.degree(a_ref)),
                                   po.start_vector(po.degree(a_ref)), TINY_EPS, 8)
    assert trace.iterations_run == 8
    assert np.abs(v - ref).sum() / np.abs(ref).sum() <= 1e-4
    # numpy W through the row scan takes the same path
    v2, _ = gpu.power_iterate(w.numpy(), params, v0)
    assert np.abs(v2 - v).sum() / np.abs(v).sum() <= 1e-5


def test_initial_vector_choices():
    gpu = _gpu()
    deg = np.array([1.0, 1.0, 2.0])
    assert np.array_equal(gpu.initial_vector(deg, "degree"), [0.25, 0.25, 0.5])
    assert np.array_equal(gpu.initial_vector(deg, "uniform"), np.full(3, 1.0 / 3.0))
    with pytest.raises(errors.ZeroDegree):
        gpu.initial_vector(np.array([1.0, 0.0]), "degree")
    with pytest.raises(errors.InvalidSpec):
        gpu.initial_vector(deg, "bogus")
    with pytest.raises(errors.InvalidSpec):
        gpu.initial_vector(deg, np.array([0.5, 0.5]))


def test_build_affinity_rejects_nonfinite():
    pts = np.zeros((4, 2))
    pts[2, 1] = np.inf
    with pytest.raises(errors.NonFiniteEntry):
        _gpu().build_affinity(DataSet(pts), GaussianRbf(1.0))


def test_generate_blobs_matches_oracle_stream():
    """gpic_generate_blobs vs the oracle's numpy restatement (Philox4x32-10,
    KAT-pinned in test_oracle_golden.py): labels exact, X to libm rounding."""
    from paper_1604_02700_b200.datasets import gaussian_blobs as host_blobs, graded_sizes

    gpu = _gpu()
    for n, d, k, seed in ((1001, 3, 3, 0), (5000, 64, 10, 7), (777, 1, 2, 2**40 + 5)):
        x, lab = gpu.generate_blobs(n, d, k, seed=seed)
        host = host_blobs(n, d, k, seed=seed)
        rng = np.random.default_rng(seed)
        c = rng.standard_normal((k, d))
        c = c / np.linalg.norm(c, axis=1, keepdims=True) * 40.0
        ref_x, ref_lab = po.device_blobs(c, graded_sizes(n, k), seed, 1.0, 8.0)
        xs = x.cpu().numpy()
        assert np.array_equal(lab.cpu().numpy(), ref_lab)
        assert np.array_equal(ref_lab, host.labels)
        assert np.abs(xs - ref_x).max() <= 1e-12 * np.abs(ref_x).max()
        x2, _ = gpu.generate_blobs(n, d, k, seed=seed)
        assert np.array_equal(x2.cpu().numpy(), xs)


def test_cluster_points_on_generated_data():
    """Device-generated X clusters exactly like the same X passed from the host."""
    from paper_1604_02700_b200 import KernelConfig, adjusted_rand_index, contingency

    gpu = _gpu()
    x, lab = gpu.generate_blobs(20000, 32, 5, seed=1)
    kind = GaussianRbf(np.sqrt(32) / 2)
    params = PicParams(k=5)
    l1, v1, t1, _ = gpu.cluster_points(x, kind, params, KernelConfig(), seed=0)
    l2, v2, t2, _ = gpu.cluster_fused(DataSet(x.cpu().numpy()), kind, params, KernelConfig(), seed=0)
    assert np.array_equal(l1, l2) and np.array_equal(v1, v2)
    assert t1.iterations_run == t2.iterations_run
    assert adjusted_rand_index(contingency(lab.cpu().numpy(), l1)) == 1.0
    with pytest.raises(errors.InvalidSpec):
        gpu.cluster_points(x.float(), kind, params)
