#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "parent or kernel_variants or test_apply_parity or spheroid" > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02o_pytest.log; tail -2 gpurun_out/r02o_pytest.log
for C in cfg2 cfg3; do timeout 900 python tools/prof_apply.py $C 5 > gpurun_out/r02o_$C.log 2>&1; tail -1 gpurun_out/r02o_$C.log; done
timeout 3000 python tools/emulate_ranks.py cfg5 8 --steps 3 > gpurun_out/r02o_cfg5_w8.json 2> gpurun_out/r02o_cfg5_w8.err; echo "cfg5 rc=$?"; tail -3 gpurun_out/r02o_cfg5_w8.err
