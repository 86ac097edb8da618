"""CSV I/O (data.py:81-138 of the reference): round trips, the reference's
errors with 1-based line numbers, and the fast path agreeing with the line
loop bit for bit."""

import numpy as np
import pytest

from paper_1604_02700_b200 import DataSet, errors, load_csv, write_csv, write_vector_csv
from paper_1604_02700_b200.data import _load_csv_lines


def test_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((500, 7)) * 10.0 ** rng.integers(-30, 30, (500, 7))
    lab = rng.integers(0, 4, 500)
    lab[:4] = [0, 1, 2, 3]
    f = tmp_path / "x.csv"
    write_csv(DataSet(pts, lab), f)
    d = load_csv(f, has_labels=True)
    assert np.array_equal(d.points, pts) and np.array_equal(d.labels, lab)
    assert d.name == "x"
    # the fast parser and the reference loop agree bit for bit
    ref_pts, ref_lab = _load_csv_lines(f, True, False)
    assert np.array_equal(ref_pts, d.points) and np.array_equal(ref_lab, d.labels)


def test_header_blank_lines_and_no_labels(tmp_path):
    f = tmp_path / "h.csv"
    f.write_text("a,b\n1.5,2\n\n3,4.25\n")
    d = load_csv(f, header=True)
    assert d.labels is None and np.array_equal(d.points, [[1.5, 2.0], [3.0, 4.25]])


@pytest.mark.parametrize("text,has_labels,exc,line", [
    ("1,2\n3,4,5\n", False, errors.RaggedRows, 2),
    ("1,2,3\n4,5\n", False, errors.RaggedRows, 2),
    ("1,2\n3,x\n", False, errors.ParseError, 2),
    ("1,2,0\n3,4,1.0\n", True, errors.ParseError, 2),
    ("1,,2\n", False, errors.ParseError, 1),
    ("\n\n", False, errors.EmptyDataSet, None),
    ("1,nan\n", False, errors.NonFiniteEntry, None),
])
def test_reference_errors(tmp_path, text, has_labels, exc, line):
    f = tmp_path / "e.csv"
    f.write_text(text)
    with pytest.raises(exc) as info:
        load_csv(f, has_labels=has_labels)
    if line is not None:
        assert info.value.line == line


def test_write_vector_csv(tmp_path):
    v = np.array([1.0 / 3.0, 2.5e-300])
    f = tmp_path / "v.csv"
    write_vector_csv(v, f)
    assert np.array_equal(np.loadtxt(f), v)
