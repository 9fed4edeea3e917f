timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "restrict" 2>&1 | tail -1
for v in new head new head; do
  if [ $v = new ]; then unset TH_LIBPATH; else export TH_LIBPATH=$PWD/_lib_ab/$v/libtrihalo_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/abs_$v.json 2>/dev/null; echo "c5 $v"; python tools/bench_brief.py gpurun_out/abs_$v.json | sed -n 1,2p
  timeout 600 python bench.py --scale 0.125 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/abs8_$v.json 2>/dev/null; echo "c5/8 $v"; python tools/bench_brief.py gpurun_out/abs8_$v.json | sed -n 2,2p
done
