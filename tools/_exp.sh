O=gpurun_out
rm -f $O/exp.log
python -m pytest tests/test_gpu_parity.py -q -x -k "ceiling" > $O/t.log 2>&1; echo t=$? >> $O/exp.log; tail -3 $O/t.log >> $O/exp.log
