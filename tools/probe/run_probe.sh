#!/bin/bash
# run on the GPU box: microbenchmarks + clocks sampled during the run
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
nvidia-smi > gpurun_out/probe_nvsmi.txt 2>&1
lscpu > gpurun_out/probe_lscpu.txt 2>&1
nproc >> gpurun_out/probe_lscpu.txt
./tools/probe/probe > gpurun_out/probe.txt 2>&1
kill $SMI
