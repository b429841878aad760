#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/prof_apply.py cfg2 2 > gpurun_out/r4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launches.csv python tools/prof_apply.py cfg2 2 > gpurun_out/r4_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"parent_kernel|cousin_kernel|leaf_fill|near_kernel|rp_combine" -s 6 -c 8 -o gpurun_out/r4_prof python tools/prof_apply.py cfg2 1 > gpurun_out/r4_ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/r4_plain.log; tail -3 gpurun_out/r4_ncu_full.log; ls -la gpurun_out/
