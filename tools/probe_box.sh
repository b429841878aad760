#!/bin/bash
mkdir -p gpurun_out
{ nproc; lscpu | head -30; free -g; nvidia-smi; ldd --version | head -1; } > gpurun_out/box_probe.txt 2>&1
./tools/fp64_peak >> gpurun_out/box_probe.txt 2>&1
./tools/fp64_peak >> gpurun_out/box_probe.txt 2>&1
cat gpurun_out/box_probe.txt
