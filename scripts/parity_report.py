"""Measured embedding error of both Gram engines against the reference (golden) and oracle."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from oracle import pic_oracle as po
from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs

G = "tests/golden/"
def pts(z):
    if "X" in z: return z["X"]
    g = json.loads(str(z["gen"])); return gaussian_blobs(g["n"], g["d"], g["k"], seed=g["seed"], sizes=g.get("sizes","graded")).points
out = {}
for case, T in (("config1", 10), ("gblobs_small", 8), ("gblobs_balanced", 5)):
    z = dict(np.load(G + case + ".npz"))
    d = DataSet(pts(z))
    for eng in ("simt", "tc"):
        lab, v, tr = cluster(d, GaussianRbf(float(z["sigma"])), PicParams(k=int(z["k"])), config=KernelConfig(affinity_impl=eng), seed=int(z["seed"]))
        _, vT, _ = cluster(d, GaussianRbf(float(z["sigma"])), PicParams(k=int(z["k"]), epsilon=5e-324, max_iterations=T), config=KernelConfig(affinity_impl=eng))
        ref = z[f"v_T{T}"]
        r = dict(labels_equal=bool(np.array_equal(lab, z["labels"])), iters=tr.iterations_run, ref_iters=int(z["iterations"]),
                 rel_l1_native=float(np.abs(v - z["v"]).sum() / np.abs(z["v"]).sum()),
                 rel_l1_forced=float(np.abs(vT - ref).sum() / np.abs(ref).sum()), T=T)
        out[f"{case}/{eng}"] = r
        print(case, eng, r, flush=True)
# a config-3-shaped case small enough for the fp64 oracle: n=8000, d=64, k=10
d = gaussian_blobs(8000, 64, 10, seed=3)
a = po.affinity(d.points, 4.0); deg = po.degree(a); w = po.normalize(a, deg); del a
ref, _, _ = po.power_iteration(w, po.start_vector(deg), 5e-324, 6)
for eng in ("simt", "tc"):
    _, v6, _ = cluster(d, GaussianRbf(4.0), PicParams(k=10, epsilon=5e-324, max_iterations=6), config=KernelConfig(affinity_impl=eng))
    e = float(np.abs(v6 - ref).sum() / np.abs(ref).sum())
    out[f"n8000_d64/{eng}"] = dict(rel_l1_forced=e, T=6)
    print("n8000 d64", eng, e, flush=True)
json.dump(out, open("gpurun_out/parity_report.json", "w"), indent=1)
