O=gpurun_out
rm -f $O/exp.log
python -m pytest tests/test_gpu_parity.py -q -x > $O/t.log 2>&1; echo t=$? >> $O/exp.log; tail -1 $O/t.log >> $O/exp.log
AMP_NO_RUN_SLOT=1 python -m pytest tests/test_gpu_parity.py -q -x -k "full_sweep_1m or ceiling or shape" > $O/t2.log 2>&1; echo t2=$? >> $O/exp.log; tail -1 $O/t2.log >> $O/exp.log
run() { echo "== $*" >> $O/exp.log; env "$@" python tools/prof_eval.py 100000000 2>&1 | tail -1 | sed 's/inner.*//' >> $O/exp.log; }
run AMP_X=0
run AMP_X=1
