#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/diag_parity.py > gpurun_out/r3_diag.log 2>&1; echo "rc=$?" >> gpurun_out/r3_diag.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -s > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err; echo "bench rc=$?" >> gpurun_out/r3_bench.err
cat gpurun_out/r3_diag.log; tail -25 gpurun_out/r3_pytest.log; cat gpurun_out/r3_bench.json; tail -5 gpurun_out/r3_bench.err
