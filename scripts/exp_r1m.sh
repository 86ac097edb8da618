#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_m.log 2>&1; echo "pytest rc=$?" >> $O/pytest_m.log
for st in packed packed16; do
  timeout 300 python bench.py --config 3 --storage $st --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gemv-reps 10 > $O/b3m_$st.log 2>&1
done
