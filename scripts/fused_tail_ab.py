"""A/B of the fused iteration kernel (GPIC_FUSED_TAIL=1, opt-in) against the
three-kernel tail (reduce + low rows + tail): embeddings, delta histories and
labels must be bitwise equal; prints the iterate-phase time of each.

    python scripts/fused_tail_ab.py [KNOB]     # parent: runs KNOB=0 and KNOB=1
                                               # (default GPIC_FUSED_TAIL; also
                                               # GPIC_TAU_IN_REDUCE)
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = ("config3", "isolated", "cfg2_packed16", "small_cosine")


def child(out):
    import torch  # noqa: F401
    from paper_1604_02700_b200 import (Cosine, DataSet, GaussianRbf, KernelConfig, PicParams,
                                       gaussian_blobs, gpu)
    from paper_1604_02700_b200.datasets import config_dataset
    res = {}
    d3 = config_dataset(3, 0)
    for name in CASES:
        if name == "config3":
            d, kind, p, cfg = d3, GaussianRbf(4.0), PicParams(k=10), KernelConfig()
        elif name == "isolated":
            rng = np.random.default_rng(1)
            pts = rng.normal(size=(3000, 16))
            pts[17] += 12.5  # ~50 from the rest: fp32 row flushes, fp64 degree ~1e-60
            d, kind, p, cfg = DataSet(pts), GaussianRbf(3.0), PicParams(k=3), KernelConfig()
        elif name == "cfg2_packed16":
            d, kind, p = config_dataset(2, 0), GaussianRbf(3.0), PicParams(k=5)
            cfg = KernelConfig(storage="packed16")
        else:
            d, kind, p, cfg = gaussian_blobs(5000, 24, 4, seed=3), Cosine(), PicParams(k=4), KernelConfig()
        labels, v, tr, ph = gpu.cluster_fused(d, kind, p, cfg, 0, timed=True)
        ts, ta, trs = [], [], []
        for _ in range(5):
            ph = gpu.cluster_fused(d, kind, p, cfg, 0, timed=True)[3]
            ts.append(ph["iterate"])
            ta.append(ph["affinity"])
            trs.append(ph["rowsum"])
        res[name + "_affinity_ms"] = np.median(ta) * 1e3
        res[name + "_rowsum_ms"] = np.median(trs) * 1e3
        res[name + "_labels"] = labels
        res[name + "_v"] = v
        res[name + "_hist"] = tr.delta_history
        res[name + "_iterate_ms"] = np.median(ts) * 1e3
    np.savez(out, **res)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1].endswith(".npz"):
        child(sys.argv[1])
        sys.exit(0)
    knob = sys.argv[1] if len(sys.argv) > 1 else "GPIC_FUSED_TAIL"
    values = sys.argv[2:] or ["0", "1"]
    outs = {}
    for flag in values:
        out = f"/tmp/tail_ab_{knob}_{flag}.npz"
        env = dict(os.environ, **{knob: flag})
        subprocess.run([sys.executable, __file__, out], check=True, env=env)
        outs[flag] = np.load(out)
    a = outs[values[0]]
    ok = True
    for flag in values[1:]:
        b = outs[flag]
        for name in CASES:
            same = all(np.array_equal(a[f"{name}_{k}"], b[f"{name}_{k}"])
                       for k in ("labels", "v", "hist"))
            ok &= same
            print(f"{name}: bitwise {'equal' if same else 'DIFFERENT'}; iterate "
                  f"{float(a[name + '_iterate_ms']):.3f} ms ({knob}={values[0]}) -> "
                  f"{float(b[name + '_iterate_ms']):.3f} ms ({knob}={flag}), "
                  f"T = {len(b[name + '_hist'])}; affinity "
                  f"{float(a[name + '_affinity_ms']):.3f} -> {float(b[name + '_affinity_ms']):.3f} ms; "
                  f"rowsum {float(a[name + '_rowsum_ms']):.3f} -> {float(b[name + '_rowsum_ms']):.3f} ms")
    sys.exit(0 if ok else 1)
