#!/bin/bash
# quick check: a pytest subset, then per-phase apply times (and setup debug) at configs
#   gpurun -- ./tools/gpu_quick.sh <tag> "<pytest -k expr or empty>" cfgA [cfgB ...]
TAG=$1; K=$2; shift 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
for CFG in "$@"; do
  IFGF_SETUP_DEBUG=1 timeout 900 python tools/prof_apply.py $CFG 5 > gpurun_out/${TAG}_${CFG}.log 2>&1
  grep -v "^templates" gpurun_out/${TAG}_${CFG}.log | tail -6
  python - <<PY
import sys; sys.path.insert(0,'.')
PY
done
