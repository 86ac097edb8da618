"""Where cluster()'s end-to-end time goes beyond the device run (config 3):
wall time of the public call vs gpic_cluster alone vs its pieces."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster  # noqa: E402
from paper_1604_02700_b200.datasets import config_dataset  # noqa: E402

d = config_dataset(3, 0)
host = torch.empty(d.points.shape, dtype=torch.float64).pin_memory()
host.numpy()[:] = d.points
dh = DataSet(host.numpy(), d.labels)
kind, params, cfg = GaussianRbf(4.0), PicParams(k=10), KernelConfig()
for _ in range(3):
    cluster(dh, kind, params, config=cfg)
torch.cuda.synchronize()
t = []
for _ in range(10):
    t0 = time.perf_counter()
    cluster(dh, kind, params, config=cfg)
    t.append(time.perf_counter() - t0)
print(f"cluster() e2e median {np.median(t) * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    cluster(dh, kind, params, config=cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(14)
