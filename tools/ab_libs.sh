#!/bin/bash
# A/B of library builds at one config: ./tools/ab_libs.sh <cfg> <applies> base <variant>...
# (variants from tools/build_variant.sh; "base" = the in-tree library)
cd $GRAFT_REPO_ROOT; CFG=$1; N=$2; shift 2
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2112_06316_b200/lib/variants/$v.so; fi
  echo "== $v"; IFGF_B200_LIB=$L timeout 600 python tools/prof_apply.py $CFG $N 2>&1 | tail -1 | cut -c1-300
done
