#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/prof_apply.py cfg2 1 > gpurun_out/r8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"parent_tc" -s 0 -c 3 -o gpurun_out/r8_prof python tools/prof_apply.py cfg2 1 > gpurun_out/r8_ncu.log 2>&1
echo rc=$?; tail -2 gpurun_out/r8_ncu.log
