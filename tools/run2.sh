#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/diag_parity.py > gpurun_out/r2_diag.log 2>&1; echo "rc=$?" >> gpurun_out/r2_diag.log
cat gpurun_out/r2_diag.log
