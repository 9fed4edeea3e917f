timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py -q -x -m gpu -k "order3 or simulated or pool_interp" 2>&1 | tail -1
for v in mbar named mbar named; do
  if [ $v = named ]; then export TH_LIBPATH=$PWD/_lib_ab/b2t2/libtrihalo_b200.so; else unset TH_LIBPATH; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/abq_$v.json 2>/dev/null; echo "c5 $v"; python tools/bench_brief.py gpurun_out/abq_$v.json | sed -n 3,3p
  timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu --no-same-level > gpurun_out/c3p_$v.json 2>/dev/null; echo "c3 $v"; python tools/bench_brief.py gpurun_out/c3p_$v.json | sed -n 3,3p
done
unset TH_LIBPATH
cmd="python bench.py --scale 0.125 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $cmd > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile3p -s 1 -c 1 -f -o gpurun_out/prof_t3p $cmd > gpurun_out/ncu_t3p.log 2>&1; tail -1 gpurun_out/ncu_t3p.log
