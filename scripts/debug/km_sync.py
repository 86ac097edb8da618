import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import _lib, gpu
L = _lib.lib()
n, k = 40000, 3
rng = np.random.default_rng(n + k)
levels = np.sort(rng.uniform(1e-6, 1e-6 + 1e-4, k))
v = rng.choice(levels, n) * (1 + 1e-3 * rng.standard_normal(n))
dev = torch.device("cuda")
vt = torch.from_numpy(v).to(dev)
first, u = gpu.kmeans_draws(n, k, 0)
scratch = torch.zeros(int(L.gpic_kmeans_scratch_bytes(n, k)), dtype=torch.uint8, device=dev)
labels = torch.full((n,), -7, dtype=torch.int64, device=dev)
ctl = gpu._new_ctl(dev)
L.gpic_kmeans1d(C.c_void_p(vt.data_ptr()), n, k, first, u.ctypes.data_as(C.c_void_p), 100, 1e-12,
                C.c_void_p(labels.data_ptr()), C.c_void_p(scratch.data_ptr()), C.c_void_p(ctl.data_ptr()), None)
torch.cuda.synchronize()
al = lambda b: (b + 255) & ~255
m = min(n, 4096)
st_off = al(n * 4) * 2 + al(n * 8) + al(64 * 8) + al(m * 4) + al((m + 1) * 8) + al(65 * (m + 1) * 4)
stats = scratch.cpu().numpy()[st_off: st_off + 64 * 8].view(np.float64)
print("per-CTA (mod 64) nsync + 1000*ph:", np.unique(stats, return_counts=True))
print("status", gpu._read_ctl(ctl, dev).status)
raw = scratch.cpu().numpy()
lab = raw[: n * 4].view(np.int32)
gpo = st_off + al(64 * 8)
words_d = raw[gpo: gpo + (776 + 2 * 65536) * 8].view(np.float64)
words_i = raw[gpo: gpo + (776 + 2 * 65536) * 8].view(np.int64)
G = 148
for buf in (0, 1):
    base = 776 + buf * 65536
    for j in range(k):
        mxs = [words_d[base + (q * 64 + j) * 4 + 2] for q in range(G)]
        mns = [words_d[base + (q * 64 + j) * 4 + 0] for q in range(G)]
        sel = lab == j
        print(f"buf {buf} j {j}: reduce mn {min(mns):.6e} mx {max(mxs):.6e} | true mn {v[sel].min():.6e} mx {v[sel].max():.6e}")
