#!/bin/bash
# Memory-safety check without compute-sanitizer (closed on the GPU pool): the
# GPU test suite against the bounds-checked build (-DAMP_BOUNDS: every
# AMP_CHECK in the kernels traps on a violation), run via gpurun.
O=gpurun_out
mkdir -p _var
make lib LIB=_var/bounds.so EXTRA="-DAMP_BOUNDS" > $O/bounds_build.log 2>&1 || { echo build failed; exit 1; }
AMP_SEARCH_LIB=_var/bounds.so timeout 1500 python -m pytest tests -m gpu -q -k "not dropin" > $O/pytest_bounds.log 2>&1
echo pytest_bounds=$?; tail -3 $O/pytest_bounds.log
echo "bounds violations: $(grep -c AMP_BOUNDS $O/pytest_bounds.log)"
