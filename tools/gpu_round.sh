#!/bin/bash
# End-of-round GPU pass: smoke, the -m gpu suite, bench lines (cfg3 default, cfg2, cfg1), the cfg3
# ncu launch list (device time + DRAM bytes per launch) and a full ncu capture of the apply
# kernels at cfg2 (cfg3's 150 GB working set defeats ncu's replay memory save/restore).
#   gpurun --timeout 4000 -- ./tools/gpu_round.sh <tag>
TAG=${1:-round}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg3 cfg2 cfg1; do
  timeout 1200 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
CMD="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-check"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_cfg3.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu list rc=$?"
CMD2="python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline --no-check"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"parent_tc|parent_cb|cousin_tc|leaf_ray|near_pair|near_list|rp_accum" \
    -c 14 -o gpurun_out/${TAG}_prof_cfg2 $CMD2 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/${TAG}_smoke.log; tail -3 gpurun_out/${TAG}_pytest.log
for c in cfg3 cfg2 cfg1; do python3 -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), d['value'], d['e2e']['value'], d.get('rel_l2_vs_reference'), d['clocks'])" 2>&1 | tail -1; done
