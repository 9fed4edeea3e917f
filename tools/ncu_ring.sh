#!/bin/bash
# ncu --set full of the slice-ring interpolation kernel:  gpurun -- 'bash tools/ncu_ring.sh <config> <NA> [extra bench args]'
mkdir -p gpurun_out
cfg=$1; na=$2; shift 2
cmd="python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-same-level $*"
TH_RING=15 TH_RING_NA=$na timeout 600 $cmd > gpurun_out/ncu_ring_plain.json 2> gpurun_out/ncu_ring_plain.err || { tail -5 gpurun_out/ncu_ring_plain.err; exit 1; }
TH_RING=15 TH_RING_NA=$na timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"ring_interp" -s 2 -c 2 -o gpurun_out/prof_ring_c$cfg -f $cmd > gpurun_out/ncu_ring.log 2>&1
tail -2 gpurun_out/ncu_ring.log
