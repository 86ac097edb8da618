#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "matrix_free or sharded or virtual" > $O/pytest_l.log 2>&1; echo "pytest rc=$?" >> $O/pytest_l.log
timeout 600 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5l.log 2>&1
GPIC_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config 3 > $O/b3l_n2.log 2>&1
GPIC_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --config 3 > $O/b3l_ref_n2.log 2>&1
