#!/bin/bash
# Profiling pass on the GPU box: launch list of one bench step + ncu --set full
# of the two dominant kernels. Outputs land in gpurun_out/ (copy summaries to profiles/).
set -x
OUT=gpurun_out
CFG=${CFG:-3}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_cfg$CFG.csv python bench.py --config $CFG --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 \
  -o $OUT/prof_gemv_cfg$CFG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline \
  --e2e-steps 0 --gemv-reps 1 > $OUT/prof_gemv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:affinity_tc_kernel -c 1 \
  -o $OUT/prof_tc_cfg2 -f python bench.py --config 2 --steps 1 --warmup 0 --no-cpu-baseline \
  --e2e-steps 0 --gemv-reps 1 > $OUT/prof_tc.log 2>&1
ls -la $OUT
