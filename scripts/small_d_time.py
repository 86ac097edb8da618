"""Affinity phase at n = 100k for small d: the SIMT difference-form engine
(d <= 8, RBF) against the tcgen05 engine just above the cut (d = 9..16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, gaussian_blobs, gpu  # noqa: E402

for d in (2, 8, 9, 16):
    g = gaussian_blobs(100_000, d, 10, seed=0)
    kind = GaussianRbf(np.sqrt(d) / 2)
    for _ in range(2):
        _, _, tr, ph = gpu.cluster_fused(g, kind, PicParams(k=10), KernelConfig(), timed=True)
    print(f"d={d:3d}: affinity {1e3 * ph['affinity']:.2f} ms, iterate {1e3 * ph['iterate']:.2f} ms "
          f"({tr.iterations_run} it)")
