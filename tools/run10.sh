#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for X in 1 2; do IFGF_B200_LIB=$PWD/paper_2112_06316_b200/lib/libexp$X.so timeout 300 python tools/prof_apply.py cfg2 5 2>&1 | tail -1 > gpurun_out/r10_exp$X.log; done
cat gpurun_out/r10_exp*.log
