#!/bin/bash
# cell-batched parent: phases at MINAVG thresholds + ncu capture of the batched kernel
TAG=$1; CFG=${2:-cfg2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in 100; do
  IFGF_SETUP_DEBUG=1 IFGF_PARENT_CB=1 IFGF_PARENT_CB_MINAVG=$m timeout 900 python tools/prof_apply.py $CFG 10 > gpurun_out/${TAG}_m$m.log 2>&1
  echo "== MINAVG=$m"; grep "cell-batched" gpurun_out/${TAG}_m$m.log; tail -1 gpurun_out/${TAG}_m$m.log | cut -c1-250
done
IFGF_PARENT_CB=1 ncu --set full --clock-control none --import-source on -k regex:"parent_cb|parent_tc" -c 6 -o gpurun_out/${TAG}_prof python tools/prof_apply.py $CFG 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?
