#!/bin/bash
# A/B of an environment switch at cfg3 (one operator per setting): ./tools/ab_cfg3.sh VAR value
cd $GRAFT_REPO_ROOT
python tools/prof_apply.py cfg3 5 | tail -1 | cut -c1-260
env $1=$2 python tools/prof_apply.py cfg3 5 | tail -1 | cut -c1-260
