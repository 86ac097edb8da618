#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_n.log 2>&1; echo "pytest rc=$?" >> $O/pytest_n.log
for st in packed packed16; do
  timeout 300 python bench.py --config 3 --storage $st --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gemv-reps 10 > $O/b3n_$st.log 2>&1
done
timeout 600 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5n.log 2>&1
