import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1604_02700_b200 import _lib, gpu, DataSet
from paper_1604_02700_b200.datasets import config_dataset
d=config_dataset(3,0); n=d.n
perm0=np.random.default_rng(5).permutation(n)
pts=d.points[perm0]; lab=d.labels[perm0]
L=_lib.lib(); dev=torch.device("cuda",0); st=torch.cuda.current_stream()
k,T=10,50; m=64
nbytes=gpu.workspace_bytes(n,m,k,T,1); work=torch.empty(nbytes,dtype=torch.uint8,device=dev)
x=torch.from_numpy(pts).to(dev); labels=torch.empty(n,dtype=torch.int64,device=dev); v=torch.empty(n,dtype=torch.float64,device=dev); hist=torch.zeros(T,dtype=torch.float64,device=dev)
first,u=gpu.kmeans_draws(n,k,0); it,cv=C.c_int32(0),C.c_int32(0); p=lambda t:C.c_void_p(t.data_ptr())
assert L.gpic_cluster(p(x),n,m,4.0,0,k,1e-5/n,T,first,u.ctypes.data_as(C.c_void_p),0,1,None,p(labels),p(v),p(hist),C.byref(it),C.byref(cv),p(work),nbytes,C.c_void_p(st.cuda_stream))==0
perm=torch.empty(n,dtype=torch.int32,device=dev); re=C.c_int32(0)
assert L.gpic_cluster_permutation(p(work),n,m,k,T,p(perm),C.byref(re),C.c_void_p(st.cuda_stream))==0
print("reordered", re.value)
pp=perm.cpu().numpy(); print("is permutation", np.array_equal(np.sort(pp), np.arange(n)))
lab2=lab[pp]; B=512; nb=-(-n//B)
print("pure blocks", sum(len(np.unique(lab2[i*B:(i+1)*B]))==1 for i in range(nb)), "of", nb)
print("first 40 labels", lab2[:40])
runs=np.flatnonzero(np.diff(lab2))+1; print("label runs", len(runs)+1)
