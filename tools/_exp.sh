O=gpurun_out
rm -f $O/exp.log
run() { echo "== $*" >> $O/exp.log; env "$@" python tools/prof_eval.py 100000000 2>&1 | tail -1 >> $O/exp.log; }
run AMP_X=0
run AMP_EST_CARVEOUT=100
run AMP_SEARCH_LIB=$PWD/variants/est_m5.so AMP_EST_CTAS_PER_SM=5 AMP_EST_CARVEOUT=100
run AMP_SEARCH_LIB=$PWD/variants/est_m5.so AMP_EST_CTAS_PER_SM=5
run AMP_SEARCH_LIB=$PWD/variants/est_m6.so AMP_EST_CTAS_PER_SM=6 AMP_EST_CARVEOUT=100
run AMP_SEARCH_LIB=$PWD/variants/est_m6.so AMP_EST_CTAS_PER_SM=6
