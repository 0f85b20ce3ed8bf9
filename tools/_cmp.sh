python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for b in 4; do AMP_DP_B=$b python tools/prof_eval.py 2000000; done
