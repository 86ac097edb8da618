#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_q.log 2>&1; echo "pytest rc=$?" >> $O/pytest_q.log
for st in packed packed16 dense; do
  timeout 200 python bench.py --config 3 --storage $st --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gemv-reps 10 > $O/b3q_$st.log 2>&1
done
timeout 200 python bench.py --config 2 --storage packed --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gemv-reps 10 > $O/b2q_packed.log 2>&1
