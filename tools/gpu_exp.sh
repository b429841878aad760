#!/bin/bash
# One experiment call: the FP64 pipe-mix probe, a GPU test subset, and env-knob A/Bs.
#   gpurun -- ./tools/gpu_exp.sh <tag> "<pytest -k expr or empty>" "<cfg>:<VAR>:<v1,v2,...>" ...
TAG=$1; K=$2; shift 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
[ -x tools/fp64_mix ] && timeout 120 ./tools/fp64_mix > gpurun_out/${TAG}_fp64_mix.json 2>&1 && cat gpurun_out/${TAG}_fp64_mix.json
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -n 2 gpurun_out/${TAG}_pytest.log
fi
for spec in "$@"; do
  IFS=: read CFG VAR VALS <<< "$spec"
  for v in ${VALS//,/ }; do
    echo "== $CFG $VAR=$v"
    env $VAR=$v timeout 900 python tools/prof_apply.py $CFG 8 > gpurun_out/${TAG}_${CFG}_${VAR}_$v.log 2>&1
    tail -n 1 gpurun_out/${TAG}_${CFG}_${VAR}_$v.log | cut -c1-400
  done
done
