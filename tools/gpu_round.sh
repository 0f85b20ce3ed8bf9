#!/bin/bash
# One GPU session: parity tests, smoke, the bench line, its launch list and
# one ncu --set full capture of a heavy k_dp_multi launch (run via gpurun).
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
python bench.py > $O/bench.log 2>&1; echo bench=$?
python bench.py --impl reference > $O/bench_ref.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-wall-time > $O/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_trie_stage -s 25 -c 1 -o $O/kdp_full -f \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-wall-time > $O/ncu_full.log 2>&1; echo full=$?
ncu -i $O/kdp_full.ncu-rep --page raw --csv > $O/kdp_full_raw.csv 2>/dev/null
ncu -i $O/kdp_full.ncu-rep --page details --csv > $O/kdp_full_details.csv 2>/dev/null
ncu -i $O/kdp_full.ncu-rep --page source --csv --print-source sass > $O/kdp_full_sass.csv 2>/dev/null
# the per-candidate kernels (thread K_place / K_est) on the bench workload:
# one launch each of the measured run (100M candidates: chunks of 64M + 36M)
ncu --set full --clock-control none --import-source on -k regex:"k_est_t|k_place_t" -s 4 -c 4 -o $O/pe_full -f \
    python tools/prof_eval.py 100000000 > $O/ncu_pe.log 2>&1; echo pe=$?
ncu -i $O/pe_full.ncu-rep --page raw --csv > $O/pe_full_raw.csv 2>/dev/null
ncu -i $O/pe_full.ncu-rep --page details --csv > $O/pe_full_details.csv 2>/dev/null
