O=gpurun_out
rm -f $O/exp.log
python -m pytest tests/test_gpu_parity.py -q -x > $O/t.log 2>&1; echo t=$? >> $O/exp.log; tail -1 $O/t.log >> $O/exp.log
AMP_CHUNK=3000000 python -m pytest tests/test_gpu_parity.py -q -x -k "full_sweep_1m or shape_kernels or memoised" > $O/t2.log 2>&1; echo t2=$? >> $O/exp.log; tail -1 $O/t2.log >> $O/exp.log
python tools/prof_eval.py 100000000 >> $O/exp.log 2>&1
AMP_DEDUP_SORT=1 python tools/prof_eval.py 100000000 >> $O/exp.log 2>&1
