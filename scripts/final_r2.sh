#!/bin/bash
# Round-2 measurement pass on one B200: default bench line, the other
# configs' lines, a warm-cache launch list and ncu --set full captures of
# the dominant kernels. Outputs in gpurun_out/ (summaries -> profiles/).
O=gpurun_out
TAG=${TAG:-r2f}
python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err
python bench.py --config 2 --steps 50 --warmup 5 > $O/bench_cfg2_$TAG.json 2>/dev/null
python bench.py --config 4 --steps 5 --warmup 3 --e2e-steps 3 > $O/bench_cfg4_$TAG.json 2>/dev/null
python bench.py --config 5 --storage none --steps 3 --warmup 3 --e2e-steps 2 > $O/bench_cfg5_$TAG.json 2>/dev/null
GPIC_LOOP_UNROLLED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  -c 400 --csv --log-file $O/launches_${TAG}_cfg3_packed.csv python bench.py --config 3 --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > /dev/null 2>&1
GPIC_LOOP_UNROLLED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sym_gemv" -s 3 -c 1 \
  -o $O/prof_${TAG}_gemv_cfg3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline \
  --e2e-steps 0 --gemv-reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"affinity_tc" -c 1 \
  -o $O/prof_${TAG}_tc_cfg3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline \
  --e2e-steps 0 --gemv-reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:affinity_tc_kernel -s 1 -c 1 \
  -o $O/prof_${TAG}_mf_cfg5 -f python bench.py --config 5 --storage none --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_${TAG}_cfg3_packed.csv > $O/launches_${TAG}_cfg3_packed.txt
for f in $O/prof_${TAG}_*.ncu-rep; do python scripts/ncu_summary.py $f; done > $O/ncu_${TAG}_summary.txt
tail -c 600 $O/bench_default_$TAG.json
