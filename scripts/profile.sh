#!/bin/bash
# Profiling pass on the GPU box: launch list of one bench step + ncu --set full
# of the dominant kernels. Outputs land in gpurun_out/ (summaries -> profiles/).
OUT=gpurun_out
TAG=${TAG:-r1}
STORAGE=${STORAGE:-packed}
GPIC_LOOP_UNROLLED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches_${TAG}_cfg3_${STORAGE}.csv python bench.py --config 3 --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 1 --gemv-reps 1 --storage $STORAGE > $OUT/launches_${TAG}.log 2>&1
GPIC_LOOP_UNROLLED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sym_gemv|gemv_bulk" -s 3 -c 1 \
  -o $OUT/prof_${TAG}_gemv_cfg3_${STORAGE} -f python bench.py --config 3 --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 --storage $STORAGE > $OUT/prof_${TAG}_gemv.log 2>&1
TCCFG=${TCCFG:-3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:affinity_tc_kernel -c 1 \
  -o $OUT/prof_${TAG}_tc_cfg${TCCFG}_${STORAGE} -f python bench.py --config $TCCFG --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 --storage $STORAGE > $OUT/prof_${TAG}_tc.log 2>&1
ls -la $OUT | tail -12
