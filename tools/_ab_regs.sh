for lib in base r112 r128 base r112 r128; do
  if [ $lib = base ]; then unset TH_LIBPATH; else export TH_LIBPATH=$PWD/_lib_ab/$lib/libtrihalo_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/abr_$lib.json 2>gpurun_out/abr_$lib.err
  echo "c5 $lib"; python tools/bench_brief.py gpurun_out/abr_$lib.json | sed -n 1,4p
  timeout 600 python bench.py --scale 0.125 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/abr8_$lib.json 2>/dev/null
  echo "c5/8 $lib"; python tools/bench_brief.py gpurun_out/abr8_$lib.json | sed -n 3,3p
done
