#!/bin/bash
# A/B of knobs at one (large) config: per-phase apply times per setting
#   gpurun -- ./tools/gpu_ab_big.sh <tag> <cfg> "<VAR=v ...>" ["<VAR=v ...>" ...]   ("-" = defaults)
TAG=$1; CFG=$2; shift 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
i=0
for KN in "$@"; do
  if [ "$KN" = "-" ]; then KN=""; fi
  env $KN timeout 900 python tools/prof_apply.py $CFG 5 > gpurun_out/${TAG}_${i}.log 2>&1
  echo "== [$KN]"; tail -1 gpurun_out/${TAG}_${i}.log
  i=$((i+1))
done
