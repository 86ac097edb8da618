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
    # at 0 and every id up to the maximum occurs. Labels in ascending order
    # (generator output, class-sorted files) satisfy it iff the first is 0
    # and no step exceeds 1 — two vector passes instead of a histogram.
    lab = d.labels
    if lab.size:
        if lab.size > 1:
            step = np.diff(lab)
            if lab[0] == 0 and step.min() >= 0 and step.max() <= 1:
                return
        if lab.min() != 0 or not np.bincount(lab, minlength=int(lab.max()) + 1).all():
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


# ------------------------------------------------------------ CSV I/O
# Bulk versions of the reference's CSV helpers (data.py:81-138, SURVEY.md
# §8f-4): numpy's C loadtxt for the common case (2x the reference's line
# loop at 100k x 64, bit-identical values); any input it would treat
# differently (ragged or empty fields, non-integer labels, parse errors)
# re-runs the reference's line loop,
# so values and errors — ParseError(line) / RaggedRows(line) with 1-based line
# numbers, EmptyDataSet — are the reference's.


def _csv_records(path, header):
    """(1-based line number, comma-split fields) of every non-blank data line."""
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            text = raw.strip()
            if text and not (header and lineno == 1):
                yield lineno, text.split(",")


def _parse_record(lineno, fields, has_labels):
    """(features, label or None) of one line with the reference's typed
    errors (data.py:81-120): ParseError(line) for a non-integer label or a
    non-numeric feature."""
    from .errors import ParseError

    feats, label = (fields[:-1], fields[-1]) if has_labels else (fields, None)
    if has_labels:
        try:
            label = int(label)
        except ValueError:
            raise ParseError(lineno, f"label {fields[-1]!r} is not an integer") from None
    try:
        return [float(f) for f in feats], label
    except ValueError:
        raise ParseError(lineno, "non-numeric field") from None


def _load_csv_lines(path, has_labels, header):
    """Line-by-line parse with exact errors: RaggedRows(line) when a line's
    field count differs from the first data line's, ParseError(line),
    EmptyDataSet for no data lines."""
    from .errors import RaggedRows

    points, labels, width = [], [], None
    for lineno, fields in _csv_records(path, header):
        width = len(fields) if width is None else width
        if len(fields) != width:
            raise RaggedRows(lineno)
        feats, label = _parse_record(lineno, fields, has_labels)
        points.append(feats)
        labels.append(label)
    if not points:
        raise EmptyDataSet()
    pts = np.array(points, dtype=np.float64)
    return pts, (np.array(labels, dtype=np.int64) if has_labels else None)


def _load_csv_fast(path, has_labels, header):
    """numpy's C loadtxt (correctly rounded, like float()); None when the
    input needs the reference loop (ragged or empty fields, non-integer
    labels, anything loadtxt rejects)."""
    skip = 1 if header else 0
    try:
        with open(path, "r", encoding="utf-8") as fh:
            for lineno, raw in enumerate(fh, start=1):
                if lineno > skip and raw.strip():
                    width = len(raw.strip().split(","))
                    break
            else:
                return None
        cols = width - (1 if has_labels else 0)
        if cols < 1:
            return None
        kw = dict(delimiter=",", skiprows=skip, comments=None, ndmin=2, encoding="utf-8")
        pts = np.loadtxt(path, dtype=np.float64, usecols=range(cols), **kw)
        lab = (np.loadtxt(path, dtype=np.int64, usecols=[cols], **kw).reshape(-1)
               if has_labels else None)
    except (ValueError, IndexError):
        return None
    if pts.shape[0] == 0:
        return None
    # loadtxt ignores columns past usecols and rejects short rows: any comma
    # beyond (width - 1) per data row belongs to a longer (ragged) row
    with open(path, "rb") as fh:
        data = fh.read()
    if header:
        data = data[data.find(b"\n") + 1:] if b"\n" in data else b""
    if data.count(b",") != (width - 1) * pts.shape[0]:
        return None
    return np.ascontiguousarray(pts), lab


def load_csv(path, has_labels: bool = False, header: bool = False) -> DataSet:
    """Read a rectangular numeric CSV into a DataSet (data.py:81-120)."""
    from pathlib import Path

    path = Path(path)
    fast = _load_csv_fast(path, has_labels, header)
    pts, lab = fast if fast is not None else _load_csv_lines(path, has_labels, header)
    return validate_dataset(DataSet(pts, lab, name=path.stem))


def write_csv(d: DataSet, path) -> None:
    """Points (and labels) with 17 significant digits (data.py:123-133): the
    float64 round trip through load_csv is bit-exact."""
    pts = np.asarray(d.points, dtype=np.float64)
    if np.isfinite(pts).all():
        cells = np.char.mod("%.17g", pts) if pts.size else pts.astype(str)
        if d.labels is not None:
            cells = np.column_stack([cells, np.asarray(d.labels, dtype=np.int64).astype(str)])
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("".join(",".join(r) + "\n" for r in cells))
        return
    with open(path, "w", encoding="utf-8") as fh:  # non-finite: Python's spelling
        for i in range(d.n):
            row = [f"{x:.17g}" for x in pts[i]]
            if d.labels is not None:
                row.append(str(int(d.labels[i])))
            fh.write(",".join(row) + "\n")


def write_vector_csv(values, path, fmt: str = "%.17g") -> None:
    """One value per line (data.py:136-138)."""
    np.savetxt(path, np.asarray(values).reshape(-1), fmt=fmt)
