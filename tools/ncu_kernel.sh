#!/bin/bash
# Full ncu capture of the launches of one kernel family during one cfg apply (after a plain run).
#   gpurun --timeout 1200 -- ./tools/ncu_kernel.sh <tag> <regex> [count] [cfg]
TAG=$1; RX=$2; C=${3:-3}; CFG=${4:-cfg2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
${SCRIPT:-python tools/prof_apply.py} $CFG 1 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RX" -c $C -o gpurun_out/${TAG}_prof ${SCRIPT:-python tools/prof_apply.py} $CFG 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?; tail -2 gpurun_out/${TAG}_ncu.log
