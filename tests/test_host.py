"""CPU-only tests: host logic, parameter records, and the C ABI surface."""

import ctypes
import pathlib
import re

import numpy as np
import pytest

from paper_1604_02700_b200 import (
    DataSet,
    GaussianRbf,
    KernelConfig,
    KMeansParams,
    PicParams,
    adjusted_rand_index,
    blobs_2d,
    cluster,
    contingency,
    errors,
    gaussian_blobs,
    jaccard_index,
    plan_rows,
    validate_dataset,
)
from paper_1604_02700_b200 import _lib
from paper_1604_02700_b200.datasets import graded_sizes

ROOT = pathlib.Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "gpic.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gpic_[a-z0-9_]+)\s*\(", text)))


class TestABI:
    def test_library_exports_every_declared_symbol(self):
        lib = ctypes.CDLL(str(_lib.LIB_PATH))
        names = header_functions()
        assert len(names) >= 15
        for name in names:
            assert hasattr(lib, name), f"{name} declared in gpic.h but not exported"

    def test_binding_covers_header(self):
        assert set(header_functions()) == set(_lib.SIGNATURES)

    def test_host_only_entry_points(self):
        L = _lib.lib()
        assert L.gpic_version().decode().endswith("sm_100a")
        assert L.gpic_affinity_pitch(100_000) == 100_000
        assert L.gpic_affinity_pitch(1000) == 1024
        assert L.gpic_feature_pitch(2) == 64 and L.gpic_feature_pitch(64) == 64
        assert L.gpic_feature_pitch(65) == 128
        assert L.gpic_row_pad(1000) % 128 == 0 and L.gpic_row_pad(1000) >= 1000 + 127
        ws = L.gpic_workspace_bytes(100_000, 64, 10, 100_000, 50)
        assert 0 < ws < 2 * 1024**3  # scratch only; A (40 GB) is separate
        assert L.gpic_workspace_bytes(0, 64, 10, 0, 50) == -1
        assert ctypes.sizeof(_lib.Ctl) == 256

    def test_status_mapping(self):
        ctl = _lib.Ctl()
        ctl.err_index = 7
        with pytest.raises(errors.ZeroDegree) as e:
            _lib.raise_for(_lib.GPIC_E_ZERO_DEGREE, ctl)
        assert e.value.index == 7
        ctl.err_index = 3 * 5 + 2
        with pytest.raises(errors.NonFiniteEntry) as e:
            _lib.raise_for(_lib.GPIC_E_NONFINITE, ctl, d=5)
        assert (e.value.row, e.value.col) == (3, 2)
        with pytest.raises(errors.NonPositiveTau):
            _lib.raise_for(_lib.GPIC_E_NONPOS_TAU, ctl)
        with pytest.raises(errors.InvalidSpec):
            _lib.raise_for(_lib.GPIC_E_INVALID)
        with pytest.raises(errors.DeviceError):
            _lib.raise_for(_lib.GPIC_E_CUDA)
        _lib.raise_for(_lib.GPIC_OK)


class TestParams:
    def test_rbf_sigma(self):
        with pytest.raises(errors.InvalidSpec):
            GaussianRbf(-1.0)
        with pytest.raises(errors.InvalidSpec):
            GaussianRbf(0.0)

    def test_pic_params(self):
        with pytest.raises(errors.InvalidSpec):
            PicParams(k=1)
        with pytest.raises(errors.InvalidSpec):
            PicParams(k=2, epsilon=0.0)
        with pytest.raises(errors.InvalidSpec):
            PicParams(k=2, max_iterations=0)
        assert PicParams(k=2).resolved_epsilon(1000) == 1e-5 / 1000
        assert PicParams(k=2, epsilon=1e-3).resolved_epsilon(1000) == 1e-3  # not divided by n

    def test_kmeans_params(self):
        with pytest.raises(errors.InvalidSpec):
            KMeansParams(k=1)

    def test_kernel_config(self):
        with pytest.raises(errors.InvalidSpec):
            KernelConfig(p=0)
        with pytest.raises(errors.InvalidSpec):
            KernelConfig(affinity_impl="triton")
        c = KernelConfig(p=1, chunk_rows=100, memory_budget_bytes=1000)
        with pytest.raises(errors.InvalidSpec):
            c.resolved_chunk_rows(10)
        assert KernelConfig(memory_budget_bytes=8 * 10 * 4).resolved_chunk_rows(10) == 4

    @pytest.mark.parametrize("n", [1, 5, 17, 100, 100_000])
    @pytest.mark.parametrize("p", [1, 2, 4, 8])
    def test_plan_rows(self, n, p):
        ranges = list(plan_rows(n, p))
        assert ranges[0][0] == 0 and ranges[-1][1] == n and len(ranges) <= p
        for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
            assert a1 == b0 and a0 < a1

    def test_no_cpu_fallback(self):
        import torch

        import paper_1604_02700_b200 as pkg

        assert pkg.gpu.cluster is pkg.k_affinity.__globals__["cluster"]
        if torch.cuda.is_available():
            pytest.skip("checks the no-device behaviour")
        with pytest.raises(errors.DeviceError):
            cluster(DataSet(np.ones((4, 2))), GaussianRbf(1.0), PicParams(k=2))
        with pytest.raises(errors.DeviceError):
            pkg.kmeans_1d(np.ones(5), KMeansParams(k=2))

    def test_unknown_backend(self):
        d = DataSet(np.ones((3, 2)))
        with pytest.raises(errors.InvalidSpec):
            cluster(d, GaussianRbf(1.0), PicParams(k=2), backend="serial")


class TestData:
    def test_validate(self):
        with pytest.raises(errors.EmptyDataSet):
            validate_dataset(DataSet(np.zeros((0, 2))))
        bad = np.ones((4, 3))
        bad[2, 1] = np.inf
        with pytest.raises(errors.NonFiniteEntry) as e:
            validate_dataset(DataSet(bad))
        assert (e.value.row, e.value.col) == (2, 1)
        with pytest.raises(errors.LabelLengthMismatch):
            validate_dataset(DataSet(np.ones((3, 2)), labels=np.array([0, 1])))
        with pytest.raises(errors.DataError):
            validate_dataset(DataSet(np.ones((3, 2)), labels=np.array([0, 2, 2])))

    def test_coercion(self):
        d = DataSet([[1, 2], [3, 4]])
        assert d.points.dtype == np.float64 and d.points.flags.c_contiguous
        assert d.n == 2 and d.m == 2

    def test_generators(self):
        d = gaussian_blobs(1000, 8, 4, seed=3)
        assert d.points.shape == (1000, 8)
        assert np.array_equal(np.bincount(d.labels), graded_sizes(1000, 4))
        assert np.array_equal(gaussian_blobs(1000, 8, 4, seed=3).points, d.points)
        b = blobs_2d(10, components=3, noise=0.0)
        assert np.array_equal(np.bincount(b.labels), [4, 3, 3])


class TestValidation:
    def test_ari_identical_and_permuted(self):
        t = np.array([0, 0, 1, 1, 2, 2])
        assert adjusted_rand_index(contingency(t, t)) == 1.0
        assert adjusted_rand_index(contingency(t, 2 - t)) == 1.0
        assert jaccard_index(contingency(t, t)) == 1.0

    def test_too_few(self):
        with pytest.raises(errors.TooFewPoints):
            adjusted_rand_index(contingency([0], [0]))
        with pytest.raises(errors.LengthMismatch):
            contingency([0, 1], [0])


def test_engine_routing_rule():
    """gpic_engine_for is host-only logic: d <= 8 RBF and large spreads go
    to the SIMT difference form (fp16 tiles then become fp32 packed tiles),
    matrix-free stays on tcgen05."""
    from paper_1604_02700_b200 import _lib

    L = _lib.lib()
    TC, SIMT = _lib.AFFINITY_TC, _lib.AFFINITY_SIMT
    rbf, cos = _lib.KIND_RBF, _lib.KIND_COSINE
    # config 3: R^2 / 2 sigma^2 = 64 -> tensor cores
    assert L.gpic_engine_for(rbf, 64, 4.0, 64.0 * 32.0, TC, _lib.STORAGE_PACKED) == TC
    # R / sigma = 100 -> SIMT difference form for stored fp32 A
    assert L.gpic_engine_for(rbf, 64, 1.0, 1e4, TC, _lib.STORAGE_PACKED) == SIMT
    assert L.gpic_engine_for(rbf, 64, 1.0, 1e4, TC, _lib.STORAGE_DENSE) == SIMT
    assert L.gpic_engine_for(rbf, 64, 1.0, 1e4, TC, _lib.STORAGE_NONE) == TC
    assert L.gpic_engine_for(rbf, 64, 1.0, 1e4, TC, _lib.STORAGE_PACKED16) == SIMT
    assert L.gpic_engine_for(rbf, 64, 4.0, 64.0 * 32.0, TC, _lib.STORAGE_PACKED16) == TC
    assert L.gpic_engine_for(rbf, 4, 4.0, 1.0, TC, _lib.STORAGE_PACKED) == SIMT
    assert L.gpic_engine_for(cos, 64, 1.0, 1e9, TC, _lib.STORAGE_PACKED) == TC
    assert L.gpic_engine_for(rbf, 700, 4.0, 1.0, TC, _lib.STORAGE_PACKED) == SIMT
