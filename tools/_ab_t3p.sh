TH_TILE3P=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "order3 or pool_interp" 2>&1 | tail -1
for v in base na5 na6 na7 base na5 na6 na7; do
  unset TH_LIBPATH; export TH_TILE3P=1
  if [ $v = base ]; then export TH_TILE3P=0; elif [ $v != na7 ]; then export TH_LIBPATH=$PWD/_lib_ab/$v/libtrihalo_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/abp_$v.json 2>gpurun_out/abp_$v.err
  echo "c5 $v"; python tools/bench_brief.py gpurun_out/abp_$v.json | sed -n 3,3p
  timeout 600 python bench.py --scale 0.125 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/abp8_$v.json 2>/dev/null
  echo "c5/8 $v"; python tools/bench_brief.py gpurun_out/abp8_$v.json | sed -n 3,3p
done
