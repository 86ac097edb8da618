#!/bin/bash
# Epilogue ablations of the packed affinity kernel (config 3), timed by ncu
# (kernel duration only; results are garbage on purpose for a != 0).
# bits: 1 no column-degree reads, 2 no TMA store, 4 no staging/store,
#       8 no exp (raw Gram), 12 = 4|8
for a in ${ABL:-0 1 2 3 4 8 12}; do
  GPIC_TC_ABLATE=$a timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:affinity_tc_kernel -c 2 --csv python bench.py --no-cpu-baseline --steps 1 --warmup 0 \
    --e2e-steps 0 --gemv-reps 1 2>/dev/null | grep gpu__time_duration | tail -1 | \
    awk -F'","' -v a=$a '{print "ablate", a, $(NF)}'
done
