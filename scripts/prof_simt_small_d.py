import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, gaussian_blobs, gpu
g = gaussian_blobs(100_000, 2, 10, seed=0)
gpu.cluster_fused(g, GaussianRbf(np.sqrt(2) / 2), PicParams(k=10, max_iterations=3), KernelConfig())
