"""Per-phase device time of one config (gpic_cluster_timed, CUDA events) for
env variants: python scripts/phase_ab.py [CFG=3] "VAR=a" "VAR=b" ..."""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, gpu  # noqa: E402
from paper_1604_02700_b200.datasets import CONFIGS, config_dataset  # noqa: E402

cfg = int(os.environ.get("CFG", "3"))
storage = os.environ.get("STORAGE", "packed")
c = CONFIGS[cfg]
d = config_dataset(cfg, 0)
if os.environ.get("SHUFFLE") == "1":  # the same points in random order
    from paper_1604_02700_b200 import DataSet
    import numpy as np
    d = DataSet(d.points[np.random.default_rng(5).permutation(d.n)])
for variant in sys.argv[1:] or ["NONE=0"]:
    for kv in variant.split(","):
        key, val = kv.split("=")
        os.environ[key] = val
    runs = []
    for _ in range(12):
        _, _, tr, ph = gpu.cluster_fused(d, GaussianRbf(c["sigma"]), PicParams(k=c["k"]),
                                         KernelConfig(storage=storage), seed=0, timed=True)
        runs.append(ph)
    med = {k: statistics.median(r[k] for r in runs[2:]) * 1e3 for k in runs[0]}
    print(f"{variant:36s} " + " ".join(f"{k} {v:.3f}" for k, v in med.items()) +
          f"  total {sum(med.values()):.3f} ms  T={tr.iterations_run}")
