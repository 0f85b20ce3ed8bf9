#!/bin/bash
# Quick GPU iteration: parity tests, then a short bench (no CPU / dense legs)
# and its launch list (run via gpurun).
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $O/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-dense --no-wall-time > $O/bench_quick.log 2>&1; echo bench=$?
tail -c 3000 $O/bench_quick.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-wall-time > $O/ncu_launch.log 2>&1; echo launches=$?
