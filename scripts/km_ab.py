"""k-means A/B on config-3-like embeddings: grid/one-CTA (k <= 64) vs the
sorted-domain variant (GPIC_KMEANS_SORTED=1); time and label equality."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from oracle import pic_oracle as po  # noqa: E402
from paper_1604_02700_b200 import KMeansParams, gpu  # noqa: E402

rng = np.random.default_rng(0)
for n, k in [(100000, 10), (20000, 5), (1000000, 50), (3000, 8)]:
    lev = np.sort(rng.uniform(0, 1e-4, k))
    v = np.abs(lev[rng.integers(0, k, n)] + 1e-7 * rng.standard_normal(n))
    vt = torch.from_numpy(v).cuda()
    res = {}
    for mode in ("0", "1"):
        os.environ["GPIC_KMEANS_SORTED"] = mode
        for _ in range(2):
            lab = gpu.kmeans_1d(vt, KMeansParams(k=k, seed=0))
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lab = gpu.kmeans_1d(vt, KMeansParams(k=k, seed=0))
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = (statistics.median(ts), lab.cpu().numpy())
    ref = po.kmeans_1d(v, k, 0) if n <= 100000 else None
    same = np.array_equal(res["0"][1], res["1"][1])
    print(f"n={n} k={k}: grid {res['0'][0]:.3f} ms, sorted {res['1'][0]:.3f} ms, same labels {same}"
          + (f", oracle equal {np.array_equal(res['1'][1], ref)}" if ref is not None else ""))
