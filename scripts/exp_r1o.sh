#!/bin/bash
O=gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_o.log 2>&1 || { echo "smoke failed rc=$?" >> $O/smoke_o.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_o.log 2>&1; echo "pytest rc=$?" >> $O/pytest_o.log
for st in packed packed16; do
  timeout 200 python bench.py --config 3 --storage $st --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gemv-reps 10 > $O/b3o_$st.log 2>&1
done
timeout 300 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5o.log 2>&1
