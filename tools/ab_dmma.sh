# A/B: tile3 order3 interpolation synthesis on DFMA (default build) vs DMMA (-DTH_AB_DMMA build in
# _lib_ab/dmma), same box, same call: parity of the DMMA build, bench lines, ncu --set full of both.
set -x
DM=$PWD/_lib_ab/dmma/libtrihalo_b200.so
TH_LIBPATH=$DM timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py -q -x -m gpu -k "order3 or simulated" 2>&1 | tail -2
for lib in base dmma base dmma; do
  if [ $lib = dmma ]; then export TH_LIBPATH=$DM; else unset TH_LIBPATH; fi
  timeout 600 python bench.py --scale 0.125 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_$lib.json 2>/dev/null
  echo "c5/8 $lib"; python tools/bench_brief.py gpurun_out/ab_$lib.json | sed -n 1,4p
  timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu --no-same-level > gpurun_out/ab3_$lib.json 2>/dev/null
  echo "c3 $lib"; python tools/bench_brief.py gpurun_out/ab3_$lib.json | sed -n 1,4p
done
unset TH_LIBPATH
cmd="python bench.py --scale 0.125 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile3_interp -s 1 -c 1 -f -o gpurun_out/ab_dfma $cmd > gpurun_out/ab_ncu1.log 2>&1
TH_LIBPATH=$DM timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile3_interp -s 1 -c 1 -f -o gpurun_out/ab_dmma $cmd > gpurun_out/ab_ncu2.log 2>&1
tail -1 gpurun_out/ab_ncu1.log gpurun_out/ab_ncu2.log
