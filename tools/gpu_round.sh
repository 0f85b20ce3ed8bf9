#!/bin/bash
# One GPU session (run via gpurun): parity tests, smoke, the bench line and
# the reference arm, the ncu launch list of the bench workload and one
# `ncu --set full` capture of its kernels (second run of tools/prof_eval.py).
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/prof_eval.py 100000000 > $O/ncu_launch.log 2>&1; echo launches=$?
# second run only: skip the first run's 6 launches of these kernels
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_trie_dp|k_trie_build|k_est_t|k_place_t" -s 6 -c 6 -o $O/pe_full -f \
    python tools/prof_eval.py 100000000 > $O/ncu_pe.log 2>&1; echo pe=$?
