#!/bin/bash
O=gpurun_out
for v in "GPIC_TC_ORDER=0" "GPIC_TC_ORDER=1" "GPIC_TC_STORE_HINT=0" "GPIC_TC_ORDER=1 GPIC_TC_STORE_HINT=0"; do
  env $v timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:affinity_tc -c 1 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > $O/p_$(echo $v | tr ' =' '__').log 2>&1
  echo "$v"; grep -E "gpu__time|dram__bytes" $O/p_$(echo $v | tr ' =' '__').log
done
