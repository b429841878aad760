#!/bin/bash
# A/B of an environment knob: tests (optional -k filter), then per-phase apply times at a config
# with the knob unset and set.   gpurun -- ./tools/gpu_ab.sh <tag> <cfg> <VAR=value> [pytest -k expr] [cfg3]
TAG=$1; CFG=$2; KNOB=$3; K=$4; BIG=$5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
IFGF_SETUP_DEBUG=1 timeout 600 python tools/prof_apply.py $CFG 10 > gpurun_out/${TAG}_A.log 2>&1
env $KNOB timeout 600 python tools/prof_apply.py $CFG 10 > gpurun_out/${TAG}_B.log 2>&1
grep -v "^templates\|^near lists" gpurun_out/${TAG}_A.log | tail -8; echo "--- $KNOB"; tail -2 gpurun_out/${TAG}_B.log
if [ -n "$BIG" ]; then
  IFGF_SETUP_DEBUG=1 timeout 900 python tools/prof_apply.py $BIG 5 > gpurun_out/${TAG}_big.log 2>&1; grep -v "^templates\|^near lists" gpurun_out/${TAG}_big.log | tail -8
fi
