"""Wall time of cluster() on P virtual ranks of one GPU (config 3 by default):
A/B of shard-path knobs, each variant in its own process (env read once)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, cluster  # noqa: E402
from paper_1604_02700_b200.datasets import CONFIGS, config_dataset  # noqa: E402

cfg_id = int(os.environ.get("CFG", "3"))
p = int(os.environ.get("P", "4"))
storage = os.environ.get("STORAGE", "packed")
c = CONFIGS[cfg_id]
d = config_dataset(cfg_id, 0)
kc = KernelConfig(p=p, virtual_ranks=True, storage=storage)
kind, params = GaussianRbf(c["sigma"]), PicParams(k=c["k"])
for _ in range(2):
    cluster(d, kind, params, config=kc, seed=0)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    lab, v, tr = cluster(d, kind, params, config=kc, seed=0)
    ts.append(time.perf_counter() - t0)
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} P={p} {storage}: median {np.median(ts)*1e3:.2f} ms "
      f"(T={tr.iterations_run})")
