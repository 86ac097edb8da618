"""Debug: whole-GPU k-means labels vs the oracle (status ignored)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from oracle import pic_oracle as po
from paper_1604_02700_b200 import _lib, gpu

L = _lib.lib()
n, k = 40000, 3
rng = np.random.default_rng(n + k)
levels = np.sort(rng.uniform(1e-6, 1e-6 + 1e-4, k))
v = rng.choice(levels, n) * (1 + 1e-3 * rng.standard_normal(n))
for mode in ("grid", "one"):
    if mode == "one":
        os.environ["GPIC_KMEANS_ONE_CTA"] = "1"
    dev = torch.device("cuda")
    vt = torch.from_numpy(v).to(dev)
    first, u = gpu.kmeans_draws(n, k, 0)
    scratch = torch.zeros(int(L.gpic_kmeans_scratch_bytes(n, k)), dtype=torch.uint8, device=dev)
    labels = torch.full((n,), -7, dtype=torch.int64, device=dev)
    ctl = gpu._new_ctl(dev)
    rc = L.gpic_kmeans1d(C.c_void_p(vt.data_ptr()), n, k, first, u.ctypes.data_as(C.c_void_p), 100,
                         1e-12, C.c_void_p(labels.data_ptr()), C.c_void_p(scratch.data_ptr()),
                         C.c_void_p(ctl.data_ptr()), None)
    torch.cuda.synchronize()
    h = gpu._read_ctl(ctl, dev)
    lab = labels.cpu().numpy()
    ref = po.kmeans_1d(v, k, 0)
    print(mode, "rc", rc, "status", h.status, "mismatch", int((lab != ref).sum()),
          "labels", np.unique(lab, return_counts=True), "ref", np.unique(ref, return_counts=True))
    for j in range(k):
        sel = lab == j
        if sel.any():
            print("  label", j, "min", v[sel].min(), "max", v[sel].max(), "first idx", np.nonzero(sel)[0][:5])

# ---- per-CTA extent records of the grid path
os.environ.pop("GPIC_KMEANS_ONE_CTA", None)
al = lambda b: (b + 255) & ~255
m = min(n, 4096)
off = al(n * 4) * 2 + al(n * 8) + al(64 * 8) + al(m * 4) + al((m + 1) * 8) + al(65 * (m + 1) * 4) + al(64 * 8)
vt = torch.from_numpy(v).to(dev)
first, u = gpu.kmeans_draws(n, k, 0)
scratch = torch.zeros(int(L.gpic_kmeans_scratch_bytes(n, k)), dtype=torch.uint8, device=dev)
labels = torch.full((n,), -7, dtype=torch.int64, device=dev)
ctl = gpu._new_ctl(dev)
L.gpic_kmeans1d(C.c_void_p(vt.data_ptr()), n, k, first, u.ctypes.data_as(C.c_void_p), 100, 1e-12,
                C.c_void_p(labels.data_ptr()), C.c_void_p(scratch.data_ptr()), C.c_void_p(ctl.data_ptr()), None)
torch.cuda.synchronize()
raw = scratch.cpu().numpy()[off:]
words_d = raw[: (776 + 2 * 65536) * 8].view(np.float64)
words_i = raw[: (776 + 2 * 65536) * 8].view(np.int64)
lab = labels.cpu().numpy()
G = 148
for buf in (0, 1):
    base = 776 + buf * 65536
    print("buffer", buf)
    for q in (0, 1, 147):
        blo, bhi = n * q // G, n * (q + 1) // G
        for j in range(k):
            r = base + (q * 64 + j) * 4
            sel = np.nonzero(lab[blo:bhi] == ref[blo:bhi] * 0 + j)[0] + blo
            print(f"  cta {q} j {j}: rec mn {words_d[r]:.6e} mni {words_i[r+1]} mx {words_d[r+2]:.6e} mxi {words_i[r+3]}"
                  f" | host mn {v[sel].min() if sel.size else None}")
st_off = al(n * 4) * 2 + al(n * 8) + al(64 * 8) + al(m * 4) + al((m + 1) * 8) + al(65 * (m + 1) * 4)
stats = scratch.cpu().numpy()[st_off: st_off + 64 * 8].view(np.float64)
print("m", stats[0], "ok", stats[1])
for j in range(k):
    print("  j", j, stats[2 + 5 * j: 7 + 5 * j])
base = 776 + 65536
bad = 0
for q in range(G):
    for j in range(k):
        r = base + (q * 64 + j) * 4
        mn, mni, mx, mxi = words_d[r], words_i[r + 1], words_d[r + 2], words_i[r + 3]
        rawlab = None
        if mxi >= 0 and mxi < n:
            pass
        if (j == 1 and mx < 6e-5) or (j == 2 and mx > 6e-5) or (j == 1 and mn < 6e-5) or (j == 2 and mn > 6e-5):
            bad += 1
            if bad < 8:
                print("anomaly cta", q, "j", j, mn, mni, mx, mxi, "range", n * q // G, n * (q + 1) // G)
print("anomalies", bad)
