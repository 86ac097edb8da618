#!/bin/bash
O=gpurun_out
for ab in 0 1; do
  GPIC_SYM_ABLATE=$ab timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 10 > $O/b3h_ab${ab}.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sym_reduce -c 20 --csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > $O/reduce_h.csv 2>&1
