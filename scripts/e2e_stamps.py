import os, sys, time, ctypes as C
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gpu, _lib
from paper_1604_02700_b200.datasets import config_dataset
d = config_dataset(3, 0)
host = torch.empty(d.points.shape, dtype=torch.float64).pin_memory(); host.numpy()[:] = d.points
dh = DataSet(host.numpy(), d.labels)
kind, params, cfg = GaussianRbf(4.0), PicParams(k=10), KernelConfig()
for _ in range(3): cluster(dh, kind, params, config=cfg)
torch.cuda.synchronize()
dev = torch.device("cuda")
# manual replica of _cluster_x with stamps
L = _lib.lib(); n, m = d.points.shape; k = 10; T = 50
st = torch.cuda.current_stream()
for rep in range(5):
    t = [time.perf_counter()]
    x = torch.from_numpy(dh.points).to(dev, non_blocking=True); t.append(time.perf_counter())
    nbytes = gpu.workspace_bytes(n, m, k, T, 1)
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev); v = torch.empty(n, dtype=torch.float64, device=dev)
    hist = torch.zeros(T, dtype=torch.float64, device=dev); t.append(time.perf_counter())
    first, u = gpu.kmeans_draws(n, k, 0); t.append(time.perf_counter())
    it, cv = C.c_int32(0), C.c_int32(0)
    p = lambda q: C.c_void_p(q.data_ptr())
    rc = L.gpic_cluster(p(x), n, m, 4.0, 0, k, 1e-5/n, T, first, u.ctypes.data_as(C.c_void_p), 0, 1, None,
                        p(labels), p(v), p(hist), C.byref(it), C.byref(cv), p(work), nbytes, C.c_void_p(st.cuda_stream))
    t.append(time.perf_counter())
    a = labels.cpu().numpy(); b = v.cpu().numpy(); c = hist[:it.value].cpu().numpy(); t.append(time.perf_counter())
    print(" ".join(f"{(t[i+1]-t[i])*1e3:.3f}" for i in range(len(t)-1)), f"total {(t[-1]-t[0])*1e3:.3f}")
