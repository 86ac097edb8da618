"""Iteration-tail variants give bitwise the same results:
* GPIC_FUSED_TAIL=1 (opt-in): reduce + low rows + tau + normalise in one
  launch (sym.cu sym_iter_tail_kernel) against the separate kernels;
* GPIC_TAU_IN_REDUCE=1 (opt-in): tau formed inside the list reduce by the
  CTAs that complete each chunk (tail.cuh tau_in_reduce) against the tail's
  own chunk sums and barrier.
The graph cache keys do not include the knobs, so each setting runs in its
own process."""

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[2])
from paper_1604_02700_b200 import Cosine, DataSet, GaussianRbf, KernelConfig, PicParams, gaussian_blobs, gpu
out = {}
rng = np.random.default_rng(1)
pts = rng.normal(size=(3000, 16))
pts[17] += 12.5  # ~50 from the rest: its fp32 row flushes, fp64 degree ~1e-60
cases = {
    "isolated": (DataSet(pts), GaussianRbf(3.0), PicParams(k=3), KernelConfig()),
    "blobs": (gaussian_blobs(20000, 32, 5, seed=0), GaussianRbf(3.0), PicParams(k=5), KernelConfig()),
    "blobs16": (gaussian_blobs(20000, 32, 5, seed=0), GaussianRbf(3.0), PicParams(k=5),
                KernelConfig(storage="packed16")),
    "cosine": (gaussian_blobs(5000, 24, 4, seed=3), Cosine(), PicParams(k=4), KernelConfig()),
}
for name, (d, kind, p, cfg) in cases.items():
    labels, v, tr, _ = gpu.cluster_fused(d, kind, p, cfg, 0)
    out[name + "_labels"], out[name + "_v"], out[name + "_hist"] = labels, v, tr.delta_history
np.savez(sys.argv[1], **out)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("knob", ["GPIC_FUSED_TAIL", "GPIC_TAU_IN_REDUCE"])
def test_tail_variants_are_bitwise_equal(tmp_path, knob):
    res = {}
    for flag in ("0", "1"):
        out = str(tmp_path / f"r{flag}.npz")
        env = dict(os.environ, **{knob: flag})
        subprocess.run([sys.executable, "-c", CHILD, out, ROOT], check=True, env=env, timeout=600)
        res[flag] = np.load(out)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res["1"][key]), key
    assert len(res["1"]["isolated_hist"]) >= 2
