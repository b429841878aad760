#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/dmma_peak > gpurun_out/r7_dmma.txt 2>&1; ./tools/fp64_peak >> gpurun_out/r7_dmma.txt 2>&1; cat gpurun_out/r7_dmma.txt
