import sys, numpy as np
sys.path.insert(0, ".")
from paper_1604_02700_b200 import gpu, GaussianRbf, KernelConfig, DataSet
from paper_1604_02700_b200.datasets import gaussian_blobs
from oracle import pic_oracle as po
d = gaussian_blobs(1500, 16, 4, seed=7)
a = gpu.k_affinity(d, GaussianRbf(2.0), KernelConfig(affinity_impl="tc"))
full = a.numpy()
ref = po.affinity(d.points, 2.0)
nz = np.abs(full - ref) > 1e-4 * ref.max()
print("bad frac", nz.mean(), "rows with bad", np.unique(np.nonzero(nz)[0])[:20], "cols", np.unique(np.nonzero(nz)[1])[:40])
r, c = np.nonzero(nz)
print("bad row%128 hist", np.bincount(r % 128, minlength=128)[:40])
print("bad col%32 hist", np.bincount(c % 32, minlength=32))
print("sample", [(int(i), int(j), float(full[i, j]), float(ref[i, j])) for i, j in list(zip(r, c))[:10]])
for r0 in (0, 32, 128, 512, 1472):
    blk = nz[r0:r0+32, :]
    cols = np.unique(np.nonzero(blk)[1])
    print("rows", r0, "..+32: bad count", int(blk.sum()), "bad cols", cols[:12], "...", cols[-4:] if cols.size else "")
print("diag-block pattern rows 0..8 x cols 0..16:")
print((full[0:8, 0:16] == 0).astype(int))
