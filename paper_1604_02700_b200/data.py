"""Input container and validation (mirrors `picluster/data.py:25-78`).

`DataSet.points` is coerced to a C-contiguous float64 (n, m) array exactly as
the reference does; the GPU path uploads it once and does its own fp64
centring and fp32 cast on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError, EmptyDataSet, LabelLengthMismatch, NonFiniteEntry


@dataclass(frozen=True)
class DataSet:
    """n points in m-dimensional space, optionally labelled (data.py:25-58)."""

    points: np.ndarray
    labels: np.ndarray | None = None
    name: str = ""

    def __post_init__(self) -> None:
        pts = np.ascontiguousarray(np.asarray(self.points, dtype=np.float64))
        if pts.ndim != 2:
            pts = np.atleast_2d(pts)
        object.__setattr__(self, "points", pts)
        if self.labels is not None:
            object.__setattr__(
                self, "labels", np.ascontiguousarray(np.asarray(self.labels, dtype=np.int64))
            )

    @property
    def n(self) -> int:
        return self.points.shape[0]

    @property
    def m(self) -> int:
        return self.points.shape[1]

    @property
    def n_classes(self) -> int:
        if self.labels is None or self.labels.size == 0:
            return 0
        return int(self.labels.max()) + 1


def check_shape(d: DataSet) -> None:
    if d.points.size == 0 or d.points.shape[0] < 1 or d.points.shape[1] < 1:
        raise EmptyDataSet()


def check_labels(d: DataSet) -> None:
    if d.labels is None:
        return
    if d.labels.shape != (d.n,):
        raise LabelLengthMismatch(d.n, int(d.labels.size))
    # np.unique(labels) == arange(k) without the O(n log n) sort: ids start
    # at 0 and every id up to the maximum occurs
    if d.labels.size and (d.labels.min() != 0 or
                          not np.bincount(d.labels, minlength=int(d.labels.max()) + 1).all()):
        raise DataError("class ids must be contiguous integers starting at 0")


def validate_dataset(d: DataSet) -> DataSet:
    """Host-side validation with the reference's error order (data.py:61-78).

    The GPU backend runs the finiteness scan on the device instead
    (gpic_prepare_points reports the first non-finite (row, col)); this host
    version is kept for API parity.
    """
    check_shape(d)
    bad = ~np.isfinite(d.points)
    if bad.any():
        r, c = np.argwhere(bad)[0]
        raise NonFiniteEntry(int(r), int(c))
    check_labels(d)
    return d
