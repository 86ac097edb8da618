"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by tests/golden/make_golden.py running the
reference package; these tests show the numpy restatement in oracle/
reproduces them, so GPU-vs-oracle parity is GPU-vs-reference parity.
"""

import hashlib
import json

import numpy as np
import pytest

from oracle import pic_oracle as po
from paper_1604_02700_b200.datasets import blobs_2d, gaussian_blobs

from conftest import GOLDEN


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _points(z):
    if "X" in z:
        return z["X"]
    g = json.loads(str(z["gen"]))
    d = gaussian_blobs(g["n"], g["d"], g["k"], seed=g["seed"], sizes=g.get("sizes", "graded"))
    assert _sha(d.points) == str(z["x_sha"]), "App-B generator drifted from the fixture"
    return d.points


def _sigma(z):
    return None if str(z.get("kind", "rbf")) == "cosine" else float(z["sigma"])


@pytest.mark.parametrize("case", ["config1", "gblobs_small", "gblobs_balanced", "cosine_blobs",
                                  "cosine_moons", "cosine_rays"])
def test_pipeline_matches_reference(golden, case):
    z = golden(case)
    x = _points(z)
    labels, v, deltas, conv = po.pic_cluster(x, _sigma(z), int(z["k"]), seed=int(z["seed"]))
    assert np.array_equal(labels, z["labels"])
    assert np.max(np.abs(v - z["v"])) <= 1e-12 * np.abs(z["v"]).max()
    assert len(deltas) == int(z["iterations"]) and bool(conv) == bool(z["converged"])
    assert np.allclose(deltas, z["deltas"], rtol=1e-9, atol=0)


@pytest.mark.parametrize("case", ["config1", "gblobs_small"])
def test_affinity_rows_and_degree_bitwise(golden, case):
    z = golden(case)
    x = _points(z)
    idx = z["a_rows_idx"]
    for r, row in zip(idx, z["a_rows"]):
        assert np.array_equal(po.rbf_rows(x, int(r), int(r) + 1, float(z["sigma"]))[0], row)
    a = po.affinity(x, float(z["sigma"]))
    assert np.allclose(po.degree(a), z["deg"], rtol=1e-14, atol=0)


def test_forced_iterations(golden):
    z = golden("config1")
    a = po.affinity(z["X"], 1.0)
    d = po.degree(a)
    w = po.normalize(a, d)
    for t in (1, 3, 10):
        v, deltas, conv = po.power_iteration(w, po.start_vector(d), 5e-324, t)
        assert len(deltas) == t and not conv
        assert np.max(np.abs(v - z[f"v_T{t}"])) <= 1e-15


def test_config1_generator_matches_reference(golden):
    z = golden("config1")
    d = blobs_2d(1000, components=3, noise=0.3, seed=0)
    assert np.array_equal(d.points, z["X"])
    assert np.array_equal(d.labels, z["truth"])


def test_kmeans_cases(golden):
    z = golden("kmeans")
    off = z["offsets"]
    for i, (k, s) in enumerate(zip(z["k"], z["seed"])):
        v = z["values"][off[i]: off[i + 1]]
        got = po.kmeans_1d(v, int(k), int(s))
        assert np.array_equal(got, z["labels"][off[i]: off[i + 1]]), f"case {i}"


def test_tree_sum_and_power_kats(golden):
    z = golden("kernels")
    pos = 0
    for ln, s in zip(z["reduce_lens"], z["reduce_sums"]):
        assert po.tree_sum(z["reduce_vals"][pos: pos + ln]) == s
        pos += ln
    v, deltas, conv = po.power_iteration(z["w8"], np.full(8, 1 / 8), 1e-6, 30)
    assert len(deltas) == int(z["it8"])
    assert np.max(np.abs(v - z["v8"])) <= 1e-15
    v, deltas, conv = po.power_iteration(np.eye(3), np.full(3, 1 / 3), 1e-8, 50)
    assert conv and len(deltas) == int(z["ident_it"]) == 2
    assert np.max(np.abs(po.matvec_threaded(z["mul_w"], z["mul_v"], 4) - z["mul_out"])) <= 1e-15


def test_error_cases():
    e = json.loads((GOLDEN / "errors.json").read_text())
    with pytest.raises(po.OracleError) as info:
        po.pic_cluster(np.array(e["zero_degree"]["points"]), e["zero_degree"]["sigma"], 2)
    assert info.value.kind == "ZeroDegree" and info.value.index == e["zero_degree"]["index"]
    bad = np.ones((5, 3))
    bad[3, 1] = np.nan
    bad[4, 0] = np.inf
    with pytest.raises(po.OracleError) as info:
        po.pic_cluster(bad, 1.0, 2)
    assert info.value.index == (e["non_finite"]["row"], e["non_finite"]["col"])
    with pytest.raises(po.OracleError):
        po.kmeans_1d(np.array([0.5, 0.5]), 3)


def test_threaded_affinity_port_is_bitwise(golden):
    z = golden("config1")
    rows = po.affinity_rows_threaded(z["X"], 100, 300, 1.0, p=4)
    assert np.array_equal(rows, po.rbf_rows(z["X"], 100, 300, 1.0))


@pytest.mark.parametrize("case", ["cosine_blobs", "cosine_moons"])
def test_cosine_rows_bitwise(golden, case):
    z = golden(case)
    for r, row in zip(z["a_rows_idx"], z["a_rows"]):
        assert np.array_equal(po.cosine_rows(z["X"], int(r), int(r) + 1)[0], row)


def test_zero_vector_error():
    e = json.loads((GOLDEN / "errors.json").read_text())["zero_vector"]
    with pytest.raises(po.OracleError) as info:
        po.pic_cluster(np.array(e["points"]), None, 2)
    assert info.value.kind == "ZeroVector" and info.value.index == e["index"]


def test_table2_generators_and_subsampler_match_reference():
    from paper_1604_02700_b200.datasets import generate, subsample_balanced

    g = json.loads((GOLDEN / "generators.json").read_text())
    assert {c["kind"] for c in g["generate"]} == {"two-moons", "three-circles", "cassine", "shapes",
                                                  "smiley", "blobs"}
    for c in g["generate"]:
        d = generate(c["kind"], c["n"], c["noise"], c["seed"])
        assert _sha(d.points) == c["points"] and _sha(d.labels) == c["labels"], c
    for c in g["subsample"]:
        kind, n, noise, seed = c["base"]
        sub = subsample_balanced(generate(kind, n, noise, seed), c["fraction"], c["seed"])
        assert _sha(sub.points) == c["points"] and _sha(sub.labels) == c["labels"]
        assert sub.name == c["name"]


def test_oracle_reproduces_reference_experiment2_runs():
    from paper_1604_02700_b200.datasets import generate, subsample_balanced

    for case in json.loads((GOLDEN / "experiment2.json").read_text()):
        d = generate(case["kind"], 45000, 0.05, 0)
        for run in case["runs"]:
            sub = subsample_balanced(d, run["fraction"], run["seed"])
            assert sub.n == run["n"]
            labels, v, deltas, conv = po.pic_cluster(sub.points, None, case["k"], seed=run["seed"])
            assert np.array_equal(labels, run["labels"]), (case["kind"], run["fraction"])
            assert np.max(np.abs(v - run["v"])) <= 1e-12 * np.max(np.abs(run["v"]))
            assert len(deltas) == run["iterations"]


def test_row_stochastic_verdict():
    """check_row_stochastic (serial.py:63-74): np.ones((2,2)) is rejected
    (test_serial.py:110-112); 1e-9 on the row sum; [0,1] with 1e-12 slack."""
    assert po.row_stochastic_violation(np.ones((2, 2)))[:2] == ("row", 0)
    assert po.row_stochastic_violation(np.eye(3)) is None
    assert po.row_stochastic_violation(np.array([[0.5, 0.5], [0.5, 0.5 + 5e-10]])) is None
    assert po.row_stochastic_violation(np.array([[0.5, 0.5], [0.5, 0.5 + 2e-9]]))[:2] == ("row", 1)
    assert po.row_stochastic_violation(np.array([[1.5, -0.5], [0.0, 1.0]])) == ("range", None, None)
    # NaN compares false everywhere, so the reference lets it through
    assert po.row_stochastic_violation(np.array([[np.nan, 0.0], [0.0, 1.0]])) is None


def test_philox_known_answers():
    """The device generator's stream (csrc/generate.cu) restated in the oracle
    reproduces the published Philox4x32-10 known-answer vectors (Random123
    kat_vectors: zero, all-ones and pi-digit counter/key)."""
    def run(c, k):
        return [int(v) for v in po.philox4x32_10(np.array([c], dtype=np.uint64), k)[0]]

    assert run([0, 0, 0, 0], 0) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert run([0xFFFFFFFF] * 4, 2**64 - 1) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert run([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
               0xA4093822 | (0x299F31D0 << 32)) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_device_blobs_restatement_statistics():
    """The restated device stream is standard normal noise around the App-B
    centres (mean/variance within sampling error), labels in blob order."""
    rng = np.random.default_rng(3)
    centers = rng.standard_normal((3, 5)) * 10
    x, lab = po.device_blobs(centers, [4000, 5000, 6001], seed=9, noise=1.0, offset=8.0)
    assert x.shape == (15001, 5) and np.array_equal(np.bincount(lab), [4000, 5000, 6001])
    z = x - centers[lab] - 8.0
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1.0) < 0.03
