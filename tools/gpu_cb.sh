#!/bin/bash
# cell-batched parent fill: parity tests, then per-phase times with IFGF_PARENT_CB unset / 1 / force
#   gpurun -- ./tools/gpu_cb.sh <tag> [cfg]
TAG=$1; CFG=${2:-cfg2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cell_batched or PARENT_CB" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -4 gpurun_out/${TAG}_pytest.log
for v in 0 1 force; do
  IFGF_SETUP_DEBUG=1 IFGF_PARENT_CB=$v timeout 900 python tools/prof_apply.py $CFG 10 > gpurun_out/${TAG}_${v}.log 2>&1
  echo "== CB=$v"; grep "cell-batched" gpurun_out/${TAG}_${v}.log; tail -1 gpurun_out/${TAG}_${v}.log | cut -c1-250
done
