#!/bin/bash
# cell-batched parent at cfg3: the CB tests, then per-phase apply times at IFGF_PARENT_CB_MINAVG thresholds
#   gpurun -- ./tools/cb_cfg3.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cell_batched or PARENT_CB" 2>&1 | tail -1
for m in 400; do
IFGF_SETUP_DEBUG=1 IFGF_PARENT_CB=1 IFGF_PARENT_CB_MINAVG=$m timeout 900 python tools/prof_apply.py cfg3 5 > gpurun_out/${1}_cfg3_m$m.log 2>&1
echo "== CB MINAVG=$m"; tail -1 gpurun_out/${1}_cfg3_m$m.log | cut -c1-260
done
