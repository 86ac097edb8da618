#!/bin/bash
# ncu --set full of one matrix-free A.v pass (config 5 shape, 1 launch)
TAG=${TAG:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:affinity_tc_kernel -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_mf -f python bench.py --config 5 --storage none --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > gpurun_out/prof_${TAG}_mf.log 2>&1
