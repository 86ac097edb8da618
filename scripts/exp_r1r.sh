#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_r.log 2>&1; echo "pytest rc=$?" >> $O/pytest_r.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r.log 2>&1
timeout 400 python bench.py > $O/bench_r.log 2>&1
timeout 200 python bench.py --config 3 --storage packed16 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_r16.log 2>&1
timeout 400 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/bench_r5.log 2>&1
timeout 200 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_r2.log 2>&1
TAG=r1r bash scripts/profile.sh
TAG=r1r bash scripts/prof_mf.sh
