O=gpurun_out
rm -f $O/exp.log
python -m pytest tests/test_gpu_parity.py -q -x -k "shape_kernels or records_only or full_sweep_1m or thread_and_warp" > $O/t.log 2>&1; echo t=$? >> $O/exp.log; tail -3 $O/t.log >> $O/exp.log
for v in "" "AMP_NO_SHAPE=1"; do
  echo "== $v" >> $O/exp.log
  env $v python tools/prof_eval.py 100000000 >> $O/exp.log 2>&1
done
