#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r5_pytest.log
timeout 600 python tools/prof_apply.py cfg2 10 > gpurun_out/r5_prof.log 2>&1
tail -3 gpurun_out/r5_pytest.log; cat gpurun_out/r5_prof.log
