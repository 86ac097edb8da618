"""Quick tcgen05-engine check: tc vs simt affinity on a few shapes (GPU box)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, gaussian_blobs
from paper_1604_02700_b200 import gpu

for (n, d, lo, hi) in [(300, 8, 0, 300), (1000, 2, 0, 1000), (3000, 64, 0, 3000), (2500, 64, 100, 2237),
                       (2000, 128, 0, 2000), (1500, 96, 0, 1500), (4000, 32, 0, 4000)]:
    ds = gaussian_blobs(n, d, 4, seed=1)
    kind = GaussianRbf(max(np.sqrt(d) / 2, 1.0))
    t0 = time.time()
    a = gpu.k_affinity(ds, kind, KernelConfig(affinity_impl="simt"), rows=(lo, hi))
    b = gpu.k_affinity(ds, kind, KernelConfig(affinity_impl="tc"), rows=(lo, hi))
    A, B = a.a.cpu().numpy(), b.a.cpu().numpy()
    da, db = a.deg.cpu().numpy(), b.deg.cpu().numpy()
    err = np.abs(A - B).max()
    print(f"n={n} d={d} rows=[{lo},{hi}) max|simt-tc|={err:.3e} amax={A.max():.3e} "
          f"deg rel={np.max(np.abs(da-db)/da):.3e} pad_ok={np.all(B[:, n:]==0)} t={time.time()-t0:.2f}s", flush=True)
