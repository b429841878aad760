#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r12_cfg2.json 2> gpurun_out/r12_cfg2.err
timeout 2400 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r12_cfg3.json 2> gpurun_out/r12_cfg3.err; echo "cfg3 rc=$?" >> gpurun_out/r12_cfg3.err
free -g > gpurun_out/r12_free.txt
python3 -c "
import json
for f in ['gpurun_out/r12_cfg2.json','gpurun_out/r12_cfg3.json']:
    try:
        d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['setup_s'], d['setup_breakdown_s'], d['phases_ms'])
    except Exception as e: print(f, 'ERR', e)
"
tail -5 gpurun_out/r12_cfg3.err
