#!/bin/bash
# Reproduces the committed profiles: bench line, ncu launch list (device time + DRAM bytes per
# launch) and one `--set full` capture of the apply kernels.  Run under gpurun:
#   gpurun --timeout 2400 -- ./tools/profile_cfg.sh <tag> [cfg]
# then: python tools/ncu_launches.py gpurun_out/<tag>_launches.csv profiles/<tag>_ncu_launches_<cfg>.json
#       python tools/ncu_summary.py gpurun_out/<tag>_prof.ncu-rep > profiles/<tag>_ncu_full_<cfg>_summary.txt
TAG=${1:-prof}; CFG=${2:-cfg2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --config $CFG --steps 20 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-check"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"parent_tc|cousin_tc|leaf_ray|near_list|rp_accum|parent_cb" \
    -c 16 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_ncu_full.log
