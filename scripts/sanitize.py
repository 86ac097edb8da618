"""Small runs of every storage mode / kind / engine for compute-sanitizer
(memcheck, racecheck, synccheck): `compute-sanitizer --tool T python
scripts/sanitize.py`. Each case is checked against the oracle labels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import pic_oracle as po  # noqa: E402
from paper_1604_02700_b200 import (  # noqa: E402
    Cosine, GaussianRbf, KernelConfig, PicParams, blobs_2d, cluster, gaussian_blobs)

which = sys.argv[1] if len(sys.argv) > 1 else "all"
d = blobs_2d(int(os.environ.get("SAN_N", "700")), components=3, noise=0.3, seed=0)
ref_labels, _, _, _ = po.pic_cluster(d.points, 1.0, 3, seed=0)
cases = [("tc", "packed"), ("tc", "dense"), ("tc", "packed16"), ("tc", "none"), ("simt", "packed"),
         ("simt", "dense")]
for engine, storage in cases:
    if which not in ("all", storage, engine, f"{engine}:{storage}"):
        continue
    labels, _, _ = cluster(d, GaussianRbf(1.0), PicParams(k=3),
                           config=KernelConfig(affinity_impl=engine, storage=storage), seed=0)
    print(engine, storage, "labels ok" if np.array_equal(labels, ref_labels) else "LABELS DIFFER")
if which in ("all", "cosine"):
    g = gaussian_blobs(900, 8, 3, seed=1)
    labels, _, _ = cluster(g, Cosine(), PicParams(k=3), seed=0)
    print("cosine", np.bincount(labels))
if which in ("all", "d128"):
    g = gaussian_blobs(1500, 100, 4, seed=2)
    labels, _, _ = cluster(g, GaussianRbf(5.0), PicParams(k=4), seed=0)
    print("d=100", np.bincount(labels))
if which in ("all", "isolated"):
    # a point ~50 from the rest: its fp32 row flushes, the fp64 degree stays
    # ~1e-60, so the tail computes its y in fp64 every iteration (lowdeg.cuh)
    rng = np.random.default_rng(1)
    pts = rng.normal(size=(1200, 16))
    pts[17] += 12.5
    from paper_1604_02700_b200 import DataSet  # noqa: E402
    for storage in ("packed", "dense"):
        labels, _, tr = cluster(DataSet(pts), GaussianRbf(3.0), PicParams(k=2),
                                config=KernelConfig(storage=storage), seed=0)
        print("isolated", storage, np.bincount(labels), tr.iterations_run)
