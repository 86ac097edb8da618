"""GPIC on B200: a drop-in for the reference `picluster` PIC API.

`cluster(dataset, kind, params, backend="gpu", config=None, seed=0)` has the
reference's signature (picluster/__init__.py:39-45) and returns the same
(labels int64[n], embedding float64[n], PicTrace) triple. The only backend
built is "gpu" — hand-written sm_100a kernels in libgpic.so behind a C ABI
(include/gpic.h), PyTorch used for device memory and streams only. The
reference's "serial"/"parallel" CPU backends are deliberately absent: there
is no CPU fallback.
"""

from . import errors
from .data import DataSet, load_csv, validate_dataset, write_csv, write_vector_csv
from .datasets import blobs_2d, config_dataset, gaussian_blobs
from .params import (
    Cosine,
    GaussianRbf,
    KernelConfig,
    KMeansParams,
    PartitionPlan,
    PicParams,
    PicTrace,
    SimilarityKind,
    plan_rows,
)
from .validation import ContingencyTable, adjusted_rand_index, contingency, jaccard_index

__version__ = "0.1.0"

BACKENDS = ("gpu",)


def _gpu():
    import importlib

    return importlib.import_module(".gpu", __name__)


def cluster(dataset, kind, params, backend="gpu", config=None, seed=0):
    """Cluster a dataset; returns (labels, embedding, trace)."""
    if backend != "gpu":
        raise errors.InvalidSpec(
            f"unknown backend {backend!r}: this build provides only the 'gpu' backend"
        )
    return _gpu().cluster(dataset, kind, params, config=config, seed=seed)


def kmeans_1d(values, params):
    return _gpu().kmeans_1d(values, params)


def __getattr__(name):
    # stage functions live in .gpu (imported lazily so CPU-only hosts can
    # import the package, e.g. for the oracle tests)
    if name in {"k_affinity", "k_rowsum", "k_normalize", "k_reduce", "k_norm", "k_multiply",
                "initial_embedding", "iterate", "power_iterate", "check_row_stochastic", "build_affinity", "degree",
                "normalize", "initial_vector", "generate_blobs", "cluster_points", "gpu"}:
        g = _gpu()
        return g if name == "gpu" else getattr(g, name)
    raise AttributeError(name)


__all__ = [
    "BACKENDS", "ContingencyTable", "Cosine", "DataSet", "GaussianRbf", "KMeansParams",
    "KernelConfig", "PartitionPlan", "PicParams", "PicTrace", "SimilarityKind",
    "adjusted_rand_index", "blobs_2d", "cluster", "config_dataset", "contingency", "errors",
    "gaussian_blobs", "jaccard_index", "k_affinity", "k_multiply", "k_norm", "k_normalize",
    "k_reduce", "k_rowsum", "kmeans_1d", "initial_embedding", "iterate", "power_iterate",
    "check_row_stochastic", "build_affinity", "degree", "normalize", "initial_vector", "plan_rows",
    "generate_blobs", "cluster_points",
    "validate_dataset", "load_csv", "write_csv", "write_vector_csv",
]
