#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_e.log 2>&1; echo "pytest rc=$?" >> $O/pytest_e.log
for sp in 1 4; do
  GPIC_SYM_SPLIT=$sp timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 10 > $O/b3e_sp${sp}.log 2>&1
done
TAG=r1e bash scripts/prof_mf.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_gemv -s 3 -c 1 \
  -o $O/prof_r1e_gemv -f python bench.py --config 3 --steps 1 --warmup 0 \
  --no-cpu-baseline --e2e-steps 0 --gemv-reps 1 > $O/prof_r1e_gemv.log 2>&1
