"""Time gpu.kmeans_1d on a config-3-like embedding (n = 100k, k = 10)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import KMeansParams, gpu
rng = np.random.default_rng(0)
n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 100000, int(sys.argv[2]) if len(sys.argv) > 2 else 10
levels = np.sort(rng.uniform(1e-6, 1e-4, k))
v = torch.from_numpy(rng.choice(levels, n) * (1 + 1e-3 * rng.standard_normal(n))).cuda()
for _ in range(3): gpu.kmeans_1d(v, KMeansParams(k=k, seed=0))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): lab = gpu.kmeans_1d(v, KMeansParams(k=k, seed=0))
e1.record(); e1.synchronize()
print(f"ctas={os.environ.get('GPIC_KMEANS_CTAS', 'all')} n={n} k={k}: {e0.elapsed_time(e1) / 20:.3f} ms per call (incl. host draws)")
