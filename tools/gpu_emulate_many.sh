#!/bin/bash
# several rank-by-rank emulations in one call: ./tools/gpu_emulate_many.sh <tag> "cfg3:2 cfg3:4 ..."
TAG=$1; LIST=$2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for CW in $LIST; do
  CFG=${CW%%:*}; W=${CW##*:}
  timeout 3000 python tools/emulate_ranks.py $CFG $W --steps 5 > gpurun_out/${TAG}_${CFG}_w${W}.json 2> gpurun_out/${TAG}_${CFG}_w${W}.err
  echo "$CFG w$W rc=$?"
  python3 -c "
import json; d=json.load(open('gpurun_out/${TAG}_${CFG}_w${W}.json'))
p=d.get('parity') or {}
print(d['ms_per_apply_max_over_ranks'], [round(r['ms_per_apply'],1) for r in d['ranks']], p.get('S_D_noRP',{}).get('S',{}).get('rel_l2_est_full'), p.get('out_rel_l2_rp_sample'))" 2>&1 | tail -2
done
