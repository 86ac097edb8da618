#!/bin/bash
# round-1 final evidence: tests, smoke, default bench, secondary benches, profiles
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/final_pytest.log 2>&1; echo "rc=$?" >> $O/final_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1
timeout 400 python bench.py > $O/final_bench.log 2>&1
timeout 200 python bench.py --config 3 --storage packed16 --steps 10 --warmup 3 --no-cpu-baseline > $O/final_bench16.log 2>&1
timeout 200 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/final_bench2.log 2>&1
timeout 400 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/final_bench4.log 2>&1
timeout 400 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/final_bench5.log 2>&1
TAG=r1f bash scripts/profile.sh
TAG=r1f bash scripts/prof_mf.sh
