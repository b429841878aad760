#!/bin/bash
# A/B of an environment knob at one config: ./tools/ab_env.sh <cfg> <applies> VAR v1 v2 ...
cd $GRAFT_REPO_ROOT; CFG=$1; N=$2; VAR=$3; shift 3
for v in "$@"; do
  echo "== $VAR=$v"; env $VAR=$v timeout 600 python tools/prof_apply.py $CFG $N 2>&1 | tail -1 | cut -c1-300
done
