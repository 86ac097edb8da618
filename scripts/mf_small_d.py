"""Matrix-free (storage none) at small d: the difference-form SIMT pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1604_02700_b200 import (  # noqa: E402
    GaussianRbf, KernelConfig, PicParams, adjusted_rand_index, contingency, gaussian_blobs, gpu)

for n, d in ((200_000, 2), (200_000, 8)):
    g = gaussian_blobs(n, d, 10, seed=0)
    kind = GaussianRbf(np.sqrt(d) / 2)
    for _ in range(2):
        lab, _, tr, ph = gpu.cluster_fused(g, kind, PicParams(k=10), KernelConfig(storage="none"),
                                           timed=True)
    print(f"n={n} d={d}: degree pass {1e3 * ph['affinity']:.1f} ms, iterate {1e3 * ph['iterate']:.1f} ms "
          f"({tr.iterations_run} it), ARI {adjusted_rand_index(contingency(g.labels, lab)):.3f}")
