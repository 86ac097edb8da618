#!/bin/bash
# round-1 experiment batch: sym matrix-free, GEMV copy shape, read ceiling
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "matrix_free or sym or work_orders or cosine or matches_reference or kats" > $O/pytest_d.log 2>&1; echo "pytest rc=$?" >> $O/pytest_d.log
timeout 300 scripts/probe/readbw 20 > $O/readbw.log 2>&1
for sp in 1 4 16; do for pol in 1 0; do
  GPIC_SYM_SPLIT=$sp GPIC_SYM_POL=$pol timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 10 > $O/b3_sp${sp}_pol${pol}.log 2>&1
done; done
timeout 600 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5_sym.log 2>&1
GPIC_MF_SYM=0 timeout 600 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5_full.log 2>&1
