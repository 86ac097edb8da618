import os, sys, statistics, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import KMeansParams, gpu
rng = np.random.default_rng(0)
for n, k in [(100000, 10), (1000000, 50), (200000, 20)]:
    lev = np.sort(rng.uniform(0, 1e-4, k)); v = np.abs(lev[rng.integers(0, k, n)] + 1e-7 * rng.standard_normal(n))
    vt = torch.from_numpy(v).cuda(); out=[]
    for G in ("16", "24", "32", "48", "64"):
        os.environ["GPIC_KMEANS_CTAS"] = G
        for _ in range(2): gpu.kmeans_1d(vt, KMeansParams(k=k, seed=0))
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); gpu.kmeans_1d(vt, KMeansParams(k=k, seed=0)); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        out.append(f"G={G}: {statistics.median(ts):.3f}")
    print(n, k, "  ".join(out))
