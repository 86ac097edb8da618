"""One full, measured run of the UNMODIFIED reference at a benchmark config.

    python scripts/reference_full_run.py --config 3 [--p 16] [--out gpurun_out/ref_full_cfg3.json]

Runs on the GPU box's host (196 GB RAM, 16 cores): the reference package
installed into baseline/_ref (bench.py's reference arm), through its own
parallel backend exactly as `picluster.parallel.cluster` composes it
(parallel.py:236-255), with per-phase perf_counter timing like
`picluster.report.run_timed` (report.py:47-99). Config 3 holds A and W in
fp64 (2 x 80 GB). It then compares labels / v / iteration count with the
committed CPU fixture (tests/golden/config3.npz, the fp64 matrix-free oracle)
— the reference itself at the headline config — and writes one JSON record.

Not part of bench.py (it takes ~10 minutes); the record is committed under
profiles/ as the measured (not extrapolated) CPU reference time. When the
host cannot hold A, W and the p row-block temporaries of k_normalize (config
3 needs ~235 GB at p = 16), the record keeps the phases that completed.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

import picluster as ref  # noqa: E402
from picluster import parallel as P  # noqa: E402

from paper_1604_02700_b200.datasets import CONFIGS, config_dataset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--p", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    d = config_dataset(args.config, seed=0)
    ds = ref.DataSet(d.points, d.labels)
    kind = ref.GaussianRbf(c["sigma"])
    params = ref.PicParams(k=c["k"])
    cfg = P.KernelConfig(p=args.p)
    t = {}
    status = "complete"
    labels = v = trace = None

    def phase(name, fn):
        t0 = time.perf_counter()
        out = fn()
        t[name] = time.perf_counter() - t0
        print(f"{name}: {t[name]:.1f} s", flush=True)
        return out

    a = phase("affinity", lambda: P.k_affinity(ds, kind, cfg))
    deg = phase("rowsum", lambda: P.k_rowsum(a, cfg))
    try:
        w = phase("normalize", lambda: P.k_normalize(a, deg, cfg))
    except MemoryError as e:  # A + W + p row-block temporaries exceed the host
        status = f"k_normalize: MemoryError ({e}); host RAM too small for A + W in fp64"
        w = None
    del a
    if w is not None:
        v0 = P.initial_embedding(deg, params, cfg)
        v, trace = phase("iterate", lambda: P.iterate(w, v0, params, cfg))
        del w
        labels = phase("kmeans", lambda: ref.kmeans_1d(v, ref.KMeansParams(k=c["k"], seed=0)))
    rec = {"config": args.config, "n": c["n"], "d": c["d"], "k": c["k"], "sigma": c["sigma"],
           "backend": f"picluster.parallel (baseline/_ref), KernelConfig(p={args.p})",
           "status": status, "phases_s": t, "total_s": sum(t.values()) if trace else None,
           "iterations": trace.iterations_run if trace else None,
           "converged": bool(trace.converged) if trace else None,
           "deltas": trace.delta_history.tolist() if trace else None,
           "host": {"os_cpu_count": os.cpu_count(),
                    "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset"),
                    "numpy": np.__version__}}
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                rec["host"]["ram_gib"] = round(int(ln.split()[1]) / 2**20, 1)
    except OSError:
        pass
    fx = ROOT / "tests" / "golden" / f"config{args.config}.npz"
    if fx.exists() and labels is not None:
        z = np.load(fx)
        rec["vs_fixture"] = {
            "labels_identical": bool(np.array_equal(labels, z["labels"].astype(np.int64))),
            "iterations_fixture": int(z["iterations"]),
            "v_rel_l1": float(np.abs(v - z["v"]).sum() / np.abs(z["v"]).sum()),
            "v_max_abs": float(np.max(np.abs(v - z["v"]))),
            "fixture": str(z["provenance"]),
        }
    out = json.dumps(rec)
    print(out, flush=True)
    if args.out:
        pathlib.Path(args.out).write_text(out + "\n")


if __name__ == "__main__":
    main()
