#!/bin/bash
# ncu --set full of the packed affinity kernel (config 3) under two ablation settings
for a in ${ABL:-0 12}; do
  GPIC_TC_ABLATE=$a timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:affinity_tc_kernel -c 1 -o gpurun_out/prof_abl${a} -f python bench.py --no-cpu-baseline \
    --steps 1 --warmup 0 --e2e-steps 0 --gemv-reps 1 > gpurun_out/prof_abl${a}.log 2>&1
done
