O=gpurun_out
rm -f $O/exp.log
python -m pytest tests/test_gpu_parity.py -q -x -k "1e9" --durations=3 > $O/t.log 2>&1; echo t=$? >> $O/exp.log; tail -5 $O/t.log >> $O/exp.log
python tools/prof_eval.py 1000000000 >> $O/exp.log 2>&1
