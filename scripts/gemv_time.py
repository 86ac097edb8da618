"""Time the packed GEMV alone (gpic_sym_matvec) on random tiles, config 3 size."""
import ctypes as C, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import _lib
L = _lib.lib()
n = 100000
nt = -(-n // 128)
ntiles = int(L.gpic_packed_tiles(n))
dev = torch.device("cuda")
tiles = torch.rand(ntiles * 128 * 128, dtype=torch.float32, device=dev)
v32 = torch.rand(int(L.gpic_vector_pitch(n)), dtype=torch.float32, device=dev)
pf = int(L.gpic_sym_partial_floats(n))
rowp = torch.empty(pf, dtype=torch.float32, device=dev)
colp = torch.empty(pf, dtype=torch.float32, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
def run():
    return L.gpic_sym_matvec(C.c_void_p(tiles.data_ptr()), n, C.c_void_p(v32.data_ptr()), C.c_void_p(rowp.data_ptr()),
                             C.c_void_p(colp.data_ptr()), None, C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream))
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [run() for _ in range(20)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"sym GEMV: {ms:.3f} ms  {ntiles*65536/ms/1e6:.0f} GB/s")
