O=gpurun_out
rm -f $O/exp.log
python tools/plan_phases.py synthetic96 > $O/ph_sparse.log 2>&1; echo a=$? >> $O/exp.log
PLAN_DENSE=1 python tools/plan_phases.py synthetic96 > $O/ph_dense.log 2>&1; echo b=$? >> $O/exp.log
