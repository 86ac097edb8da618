#!/bin/bash
O=gpurun_out
timeout 120 scripts/probe/umma_noswz > $O/umma_probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_f.log 2>&1; echo "pytest rc=$?" >> $O/pytest_f.log
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 10 > $O/b3f.log 2>&1
timeout 600 python bench.py --config 5 --storage none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --gemv-reps 3 > $O/b5f.log 2>&1
