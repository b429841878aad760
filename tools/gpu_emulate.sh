#!/bin/bash
# rank-by-rank emulation of a multi-GPU config on one B200 (tools/emulate_ranks.py)
#   gpurun -- ./tools/gpu_emulate.sh <tag> <cfg> <world> [steps]
TAG=$1; CFG=$2; W=$3; S=${4:-5}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 3000 python tools/emulate_ranks.py $CFG $W --steps $S > gpurun_out/${TAG}_emulate.json 2> gpurun_out/${TAG}_emulate.err
echo "rc=$?"; tail -5 gpurun_out/${TAG}_emulate.err; python3 -c "
import json; d=json.load(open('gpurun_out/${TAG}_emulate.json'))
print({k: d[k] for k in ['cfg','N','world','ms_per_apply_max_over_ranks','points_per_s_emulated']})
print(json.dumps(d.get('parity'), indent=0)[:1500])"
