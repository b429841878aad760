#!/bin/bash
# Full GPU pass: smoke, the whole -m gpu suite, the default bench line (cfg3).
#   gpurun --timeout 3000 -- ./tools/gpu_full.sh <tag> [bench args...]
TAG=${1:-full}; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1200 python bench.py "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_smoke.log; tail -25 gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_bench.err
python3 -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print({k: d.get(k) for k in ['value','ms_per_step','e2e','rel_l2_vs_reference','cpu_baseline','clocks','phases_ms','setup_s']})" 2>&1 | head -20
