"""Where the end-to-end time of cluster() goes at config 3 (host X in, labels out)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster
d = bench.config_dataset(3, seed=0)
host = torch.empty(d.points.shape, dtype=torch.float64).pin_memory()
host.numpy()[:] = d.points
dh = DataSet(host.numpy(), d.labels)
kind, params, cfg = GaussianRbf(4.0), PicParams(k=10), KernelConfig()
for _ in range(3): cluster(dh, kind, params, config=cfg)
torch.cuda.synchronize()
dev = torch.device("cuda")
t = []
for _ in range(10):
    t0 = time.perf_counter(); x = host.to(dev, non_blocking=True); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
print(f"H2D 51.2 MB pinned: {np.median(t)*1e3:.3f} ms ({51.2e6/np.median(t)/1e9:.1f} GB/s)")
t = []
for _ in range(10):
    t0 = time.perf_counter(); cluster(dh, kind, params, config=cfg); t.append(time.perf_counter() - t0)
print(f"cluster() end to end: {np.median(t)*1e3:.3f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): cluster(dh, kind, params, config=cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
