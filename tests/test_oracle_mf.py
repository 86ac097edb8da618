"""The fp64 matrix-free oracle (oracle/pic_mf.c) against the reference's own outputs.

The reference cannot hold A / W at the benchmark configs, so the config 3-5
fixtures come from this oracle; this module pins it to the golden vectors the
reference itself produced (tests/golden/make_golden.py,
make_config_fixtures.py): same labels and iteration counts, v within 1e-12.
CPU only.
"""

import json

import numpy as np
import pytest

from oracle import pic_mf as pm
from oracle import pic_oracle as po
from paper_1604_02700_b200.datasets import config_dataset, gaussian_blobs

from conftest import GOLDEN


def _points(z):
    if "X" in z:
        return z["X"]
    g = json.loads(str(z["gen"]))
    return gaussian_blobs(g["n"], g["d"], g["k"], seed=g["seed"], sizes=g.get("sizes", "graded")).points


def test_exp_matches_libm():
    xs = np.concatenate([np.linspace(-750, 5, 20001), [-745.13, -708.4, 0.0, -1e-300]])
    mine = np.array([pm.lib().picmf_exp(float(x)) for x in xs])
    ref = np.exp(xs)
    normal = ref > 2.3e-308
    assert np.max(np.abs(mine[normal] - ref[normal]) / np.spacing(ref[normal])) <= 1.0
    assert np.max(np.abs(mine[~normal] - ref[~normal])) <= 5e-324
    assert np.array_equal(mine == 0, ref == 0)


@pytest.mark.parametrize("case", ["config1", "gblobs_small", "gblobs_balanced", "cosine_blobs",
                                  "cosine_rays"])
def test_pipeline_matches_reference(golden, case):
    z = golden(case)
    x = _points(z)
    sigma = float(z["sigma"])
    sigma = None if sigma < 0 else sigma
    tr = pm.power_trajectory(x, sigma)
    labels = po.kmeans_1d(tr["v"], int(z["k"]), int(z["seed"]))
    assert len(tr["deltas"]) == int(z["iterations"])
    assert np.array_equal(labels, z["labels"])
    assert np.max(np.abs(tr["v"] - z["v"])) <= 1e-12 * np.max(np.abs(z["v"]))
    assert np.max(np.abs(tr["deg"] - z["deg"]) / z["deg"]) <= 1e-13
    rows = pm.rows(x, 0, x.shape[0], sigma)[z["a_rows_idx"]]
    assert np.max(np.abs(rows - z["a_rows"])) <= 2.3e-16  # exp() rounding only


def test_forced_t_states(golden):
    """A native trajectory passes through the forced-T states (test_serial.py:23)."""
    z = golden("config1")
    tr = pm.power_trajectory(z["X"], float(z["sigma"]), keep=(1, 3))
    for t in (1, 3):
        assert np.max(np.abs(tr["kept"][t] - z[f"v_T{t}"])) <= 1e-12 * np.max(z[f"v_T{t}"])


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_config_fixture_degrees(golden, c):
    """Sampled-row degrees of every committed benchmark fixture."""
    path = GOLDEN / f"config{c}.npz"
    if not path.exists():
        pytest.skip(f"{path.name} not generated")
    z = dict(np.load(path))
    n = int(z["n"])
    if c >= 4:
        pytest.skip("n too large for a quick CPU re-check (checked when generated)")
    d = config_dataset(c, seed=0)
    rows = [0, n // 3, n - 1]
    for r in rows:
        deg = pm.degree(d.points, float(z["sigma"]), r, r + 1)[0]
        assert abs(deg - float(z["deg"][r])) <= 1e-12 * deg
    assert int(z["iterations"]) == len(z["deltas"])
    assert np.array_equal(np.sort(np.unique(z["labels"])), np.arange(int(z["k"])))


def test_negligible_block_skip_is_bitwise_neutral():
    """The n = 1M fixture's block skip (pic_mf.c picmf_set_skip): block pairs
    proved below e^-70 are left out and every fp64 row sum stays bit-identical."""
    from paper_1604_02700_b200 import gaussian_blobs

    d = gaussian_blobs(8192, 24, 6, seed=3)
    x, sigma = d.points, float(np.sqrt(24) / 2)
    blocks = pm.negligible_blocks(x, sigma)
    assert blocks.fraction > 0.2  # well-separated blobs: many pairs provable
    deg = pm.degree(x, sigma)
    v = np.random.default_rng(1).random(x.shape[0])
    y = pm.matvec(x, sigma, deg, v)
    with blocks:
        assert np.array_equal(pm.degree(x, sigma), deg)
        assert np.array_equal(pm.matvec(x, sigma, deg, v), y)
