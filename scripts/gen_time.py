"""Time gpic_generate_blobs at config 5's shape (n = 1M, d = 64) against the
host generator + H2D it replaces."""
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

from paper_1604_02700_b200 import gpu
from paper_1604_02700_b200.datasets import gaussian_blobs

n, d, k = 1_000_000, 64, 50
gpu.generate_blobs(1000, d, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    x, lab = gpu.generate_blobs(n, d, k, seed=0)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"device generate n={n} d={d}: {ms:.3f} ms/call incl. centre upload, "
      f"{(8 * n * d + 8 * n) / ms / 1e6:.0f} GB/s written")
t = time.perf_counter()
h = gaussian_blobs(n, d, k, seed=0)
t1 = time.perf_counter()
xt = torch.from_numpy(h.points).cuda()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host generate {1e3 * (t1 - t):.0f} ms + H2D {1e3 * (t2 - t1):.0f} ms")
