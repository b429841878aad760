#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r9_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r9_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r9_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r9_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err; echo "bench rc=$?" >> gpurun_out/r9_bench.err
tail -3 gpurun_out/r9_pytest.log; cat gpurun_out/r9_smoke.log; cat gpurun_out/r9_bench.json | head -c 1500; tail -2 gpurun_out/r9_bench.err
