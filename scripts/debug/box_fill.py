import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import _lib, gpu
from paper_1604_02700_b200.datasets import config_dataset, CONFIGS
for cfg in (2, 3):
    c=CONFIGS[cfg]; d=config_dataset(cfg,0); n,m=d.points.shape; k=c["k"]; T=50
    L=_lib.lib(); dev=torch.device("cuda",0); st=torch.cuda.current_stream()
    nbytes=gpu.workspace_bytes(n,m,k,T,1); work=torch.empty(nbytes,dtype=torch.uint8,device=dev)
    x=torch.from_numpy(d.points).to(dev); labels=torch.empty(n,dtype=torch.int64,device=dev); v=torch.empty(n,dtype=torch.float64,device=dev); hist=torch.zeros(T,dtype=torch.float64,device=dev)
    first,u=gpu.kmeans_draws(n,k,0); it,cv=C.c_int32(0),C.c_int32(0); p=lambda t:C.c_void_p(t.data_ptr())
    assert L.gpic_cluster(p(x),n,m,c["sigma"],0,k,1e-5/n,T,first,u.ctypes.data_as(C.c_void_p),0,1,None,p(labels),p(v),p(hist),C.byref(it),C.byref(cv),p(work),nbytes,C.c_void_p(st.cuda_stream))==0
    offs=(C.c_int64*8)(); L.gpic_cluster_workspace_layout(n,m,k,T,1,offs)
    nt=int(L.gpic_packed_tiles(n)); f=work[offs[3]:offs[3]+nt*16].view(nt,16).cpu().numpy()
    stored=(f.max(1)>0); boxes=(f>0).sum()
    print(cfg, "stored tiles", stored.sum(), "boxes stored", boxes, "of", stored.sum()*16, f"fill {boxes/(stored.sum()*16):.3f}")
