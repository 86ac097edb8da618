"""torchrun worker: row-sharded PIC over real ranks (one process per rank).

GPIC_SAME_DEVICE=1 puts every rank on cuda:0 (CUDA IPC between processes
on one device) so the real-rank path can be exercised on a one-GPU box.
"""

import os
import pathlib
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs  # noqa: E402
from paper_1604_02700_b200 import sharded  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = 0 if os.environ.get("GPIC_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    d = gaussian_blobs(2500, 32, 5, seed=4)
    kind, params = GaussianRbf(float(np.sqrt(32) / 2)), PicParams(k=5)
    labels, v, trace = cluster(d, kind, params, config=KernelConfig(p=world, device=dev, storage="dense"),
                               seed=2)
    # packed symmetric shards: same labels as one rank, embedding within 1e-6
    lp, vp, tp = cluster(d, kind, params, config=KernelConfig(p=world, device=dev), seed=2)
    # matrix-free item shards of the pruned symmetric pass
    lm, vm, tm = cluster(d, kind, params, config=KernelConfig(p=world, device=dev, storage="none"),
                         seed=2)
    agree = (sharded.all_ranks_agree(labels, v) and sharded.all_ranks_agree(lp, vp)
             and sharded.all_ranks_agree(lm, vm))
    if rank == 0:
        single = cluster(d, kind, params, config=KernelConfig(device=dev, storage="dense"), seed=2)
        same = (np.array_equal(single[0], labels) and np.array_equal(single[1], v)
                and np.array_equal(single[2].delta_history, trace.delta_history))
        packed_ok = (np.array_equal(single[0], lp) and tp.iterations_run == trace.iterations_run
                     and np.abs(vp - single[1]).sum() / np.abs(single[1]).sum() <= 1e-6)
        mf_ok = (np.array_equal(single[0], lm) and tm.iterations_run == trace.iterations_run
                 and np.abs(vm - single[1]).sum() / np.abs(single[1]).sum() <= 1e-6)
        print("RANKS_AGREE", agree, flush=True)
        print("MATCHES_SINGLE", same and packed_ok and mf_ok, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
