#!/bin/bash
# large-config (cfg3 sphere, cfg4 spheroid; N = 6.3M) device + e2e apply throughput, no CPU baseline (hours)
#   gpurun --timeout 2700 -- ./tools/bench_large.sh <tag> <cfg>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-cfg3}; CFG=${2:-cfg3}
timeout 2400 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err
echo "rc=$?" >> gpurun_out/${TAG}.err
python3 -c "
import json; d=json.load(open('gpurun_out/${TAG}.json'))
print(d['value'], d['ms_per_step'], d['e2e'], d['setup_s'], d['setup_breakdown_s'], d['phases_ms'], d['clocks'])"
tail -3 gpurun_out/${TAG}.err
