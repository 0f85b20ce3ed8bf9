#!/bin/bash
# Compare library variants on the bench workload: bash tools/var_bench.sh lib1.so lib2.so ...
for L in "$@"; do
  echo "== $L"
  AMP_SEARCH_LIB=$L timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dense --no-wall-time --no-sweep --no-e2e 2>&1 | python -c "
import json,sys
d=json.loads([x for x in sys.stdin if x.startswith('{')][-1]); print(round(d['value']/1e9,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['dp_detail']['pipeline_ms_per_step'].items()}, round(d['roofline']['frac'],3))"
done
