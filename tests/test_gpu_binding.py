"""The reference-side ctypes binding of INTEGRATION.md, run verbatim.

The `picluster/gpu_backend.py` block of INTEGRATION.md is extracted and
installed next to a copy of the reference package (baseline/_ref, when the
reference is installed there) or next to a stand-in exposing the same
`errors` / `serial.PicTrace` names (this package's, name- and
attribute-compatible). A fresh interpreter then drives `gpic_cluster_host`
through a bare `ctypes.CDLL("libgpic.so")` — no torch, no package code on
the call path — on the reference's golden inputs.
"""

import json
import os
import pathlib
import re
import shutil
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from oracle import pic_oracle as po

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _stub_source():
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# picluster/gpu_backend\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its gpu_backend.py block"
    return m.group(1)


def _package(tmp: pathlib.Path) -> str:
    pkg = tmp / "picluster"
    ref = ROOT / "baseline" / "_ref" / "picluster"
    if (ref / "__init__.py").exists():
        shutil.copytree(ref, pkg)
        origin = "reference (baseline/_ref)"
    else:
        pkg.mkdir()
        (pkg / "__init__.py").write_text(textwrap.dedent("""
            from paper_1604_02700_b200 import DataSet, GaussianRbf, Cosine, PicParams
            from . import errors
        """))
        (pkg / "errors.py").write_text("from paper_1604_02700_b200.errors import *  # noqa\n")
        (pkg / "serial.py").write_text("from paper_1604_02700_b200.params import PicTrace  # noqa\n")
        origin = "stand-in (errors / PicTrace of this package)"
    (pkg / "gpu_backend.py").write_text(_stub_source())
    return origin


DRIVER = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])      # the package copy with gpu_backend.py
sys.path.insert(1, sys.argv[2])      # repo root (stand-in imports only)
import picluster
from picluster import gpu_backend as gb
golden = sys.argv[3]
out = {"lib": gb.lib._name}
for case in ("config1", "gblobs_small", "cosine_rays"):
    z = np.load(f"{golden}/{case}.npz")
    x = z["X"] if "X" in z.files else np.load(sys.argv[4] + f"/{case}.npy")
    kind = picluster.Cosine() if float(z["sigma"]) < 0 else picluster.GaussianRbf(float(z["sigma"]))
    labels, v, tr = gb.cluster(picluster.DataSet(x), kind, picluster.PicParams(k=int(z["k"])),
                               seed=int(z["seed"]))
    out[case] = dict(labels=bool(np.array_equal(labels, z["labels"])),
                     rel_l1=float(np.abs(v - z["v"]).sum() / np.abs(z["v"]).sum()),
                     dT=abs(tr.iterations_run - int(z["iterations"])),
                     dtype=[str(labels.dtype), str(v.dtype)])
z = np.load(f"{golden}/config1.npz")
v0 = np.load(sys.argv[4] + "/v0.npy")
_, v, tr = gb.cluster(picluster.DataSet(z["X"]), picluster.GaussianRbf(1.0),
                      picluster.PicParams(k=3, v0=v0, epsilon=5e-324, max_iterations=4))
out["explicit_v0"] = v.tolist()
_, v, tr = gb.cluster(picluster.DataSet(z["X"]), picluster.GaussianRbf(1.0),
                      picluster.PicParams(k=3, v0="uniform", epsilon=5e-324, max_iterations=4),
                      storage="dense")
out["uniform_v0"] = v.tolist()
errs = json.load(open(f"{golden}/errors.json"))
def err(fn):
    try:
        fn()
    except Exception as e:
        return [type(e).__name__, getattr(e, "index", None), getattr(e, "row", None),
                getattr(e, "col", None)]
    return None
out["zero_degree"] = err(lambda: gb.cluster(picluster.DataSet(np.array(errs["zero_degree"]["points"])),
                                            picluster.GaussianRbf(1.0), picluster.PicParams(k=2)))
bad = np.ones((5, 3)); bad[3, 1] = np.nan; bad[4, 0] = np.inf
class Raw:  # points as a caller hands them over (the device scan reports the first bad entry)
    points = bad
out["non_finite"] = err(lambda: gb.cluster(Raw(), picluster.GaussianRbf(1.0), picluster.PicParams(k=2)))
out["k_too_large"] = err(lambda: gb.cluster(picluster.DataSet(np.zeros((2, 2)) + [[0, 0], [1, 1]]),
                                            picluster.GaussianRbf(1.0), picluster.PicParams(k=3)))
print(json.dumps(out))
'''


def test_integration_stub_drives_gpic_cluster_host(tmp_path):
    origin = _package(tmp_path)
    aux = tmp_path / "aux"
    aux.mkdir()
    # inputs the goldens only pin by hash: regenerate them here
    from paper_1604_02700_b200 import gaussian_blobs

    g = json.loads(str(np.load(GOLDEN / "gblobs_small.npz")["gen"]))
    np.save(aux / "gblobs_small.npy", gaussian_blobs(g["n"], g["d"], g["k"], seed=g["seed"]).points)
    v0 = np.random.default_rng(3).random(1000)
    v0 /= v0.sum()
    np.save(aux / "v0.npy", v0)
    script = tmp_path / "drive.py"
    script.write_text(DRIVER)
    env = dict(os.environ, GPIC_LIB=str(ROOT / "paper_1604_02700_b200" / "libgpic.so"))
    res = subprocess.run([sys.executable, str(script), str(tmp_path), str(ROOT), str(GOLDEN),
                          str(aux)], capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    print(origin, json.dumps({k: out[k] for k in out if "v0" not in k}))
    assert out["lib"].endswith("libgpic.so")
    for case in ("config1", "gblobs_small", "cosine_rays"):
        r = out[case]
        assert r["labels"] and r["dT"] <= 2 and r["rel_l1"] <= 1e-4, (case, r)
        assert r["dtype"] == ["int64", "float64"]
    z = np.load(GOLDEN / "config1.npz")
    for key, choice in (("explicit_v0", v0), ("uniform_v0", "uniform")):
        _, ref, _, _ = po.pic_cluster(z["X"], 1.0, 3, epsilon=5e-324, max_iterations=4, v0=choice)
        got = np.array(out[key])
        assert np.abs(got - ref).sum() / np.abs(ref).sum() <= 1e-4, key
    assert out["zero_degree"][:2] == ["ZeroDegree", 2]
    assert out["non_finite"][0] == "NonFiniteEntry" and out["non_finite"][2:] == [3, 1]
    assert out["k_too_large"][0] == "KTooLarge"
