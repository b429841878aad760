#!/bin/bash
# Quick GPU iteration: parity tests, then per-phase apply times at a config.
#   gpurun --timeout 1500 -- ./tools/gpu_check.sh <tag> [cfg] [pytest -k expr]
TAG=${1:-chk}; CFG=${2:-cfg2}; K=${3:-}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -n "$K" ]; then KA=(-k "$K"); else KA=(); fi
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x "${KA[@]}" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python tools/prof_apply.py $CFG 10 > gpurun_out/${TAG}_prof.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_prof.log
