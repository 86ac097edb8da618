"""A/B timing of the packed GEMV on a real config-3 workspace (block-sparse
tiles left by one gpic_cluster run): env variants per launch.

    python scripts/gemv_ab.py "GPIC_GEMV_PREFETCH=0" "GPIC_GEMV_PREFETCH=2" ...
"""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import _lib, gpu  # noqa: E402
from paper_1604_02700_b200.datasets import CONFIGS, config_dataset  # noqa: E402

cfg = int(os.environ.get("CFG", "3"))
c = CONFIGS[cfg]
d = config_dataset(cfg, 0)
n, m, k, T = d.n, d.m, c["k"], 50
L = _lib.lib()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
nbytes = gpu.workspace_bytes(n, m, k, T, 1)
work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
x = torch.from_numpy(d.points).to(dev)
labels = torch.empty(n, dtype=torch.int64, device=dev)
v = torch.empty(n, dtype=torch.float64, device=dev)
hist = torch.zeros(T, dtype=torch.float64, device=dev)
first, u = gpu.kmeans_draws(n, k, 0)
it, cv = C.c_int32(0), C.c_int32(0)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
assert L.gpic_cluster(p(x), n, m, c["sigma"], _lib.KIND_RBF, k, 1e-5 / n, T, first,
                      u.ctypes.data_as(C.c_void_p), _lib.AFFINITY_TC, 1, None, p(labels), p(v),
                      p(hist), C.byref(it), C.byref(cv), p(work), nbytes,
                      C.c_void_p(st.cuda_stream)) == 0
offs = (C.c_int64 * 8)()
assert L.gpic_cluster_workspace_layout(n, m, k, T, 1, offs) == 0
b = work.data_ptr()
v32 = torch.zeros(int(L.gpic_vector_pitch(n)), dtype=torch.float32, device=dev)
v32[:n] = v.float()
y = torch.empty(n, dtype=torch.float64, device=dev)
ones = torch.ones(n, dtype=torch.float64, device=dev)


def launch():
    return L.gpic_sym_matvec_sparse(C.c_void_p(b + offs[0]), 0, n, p(v32), C.c_void_p(b + offs[1]),
                                    C.c_void_p(b + offs[2]), p(ones), p(y), C.c_void_p(b + offs[3]),
                                    C.c_void_p(b + offs[4]), C.c_void_p(st.cuda_stream))


ref = None
for variant in sys.argv[1:] or ["GPIC_GEMV_PREFETCH=2"]:
    for kv in variant.split(","):
        key, val = kv.split("=")
        os.environ[key] = val
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            launch()
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 10)
    yy = y.clone()
    if ref is None:
        ref = yy
    same = bool(torch.equal(yy, ref))
    print(f"{variant:40s} median {statistics.median(times):.4f} ms  min {min(times):.4f}  bitwise-same {same}")
