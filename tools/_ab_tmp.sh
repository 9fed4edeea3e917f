timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_guards.py -k "restrict or guards or repeated" 2>&1 | tail -2
for rep in 1 2; do
for tag in tree own2; do
  if [ $tag = tree ]; then unset TH_LIBPATH; else export TH_LIBPATH=$PWD/_lib_ab/$tag/libtrihalo_b200.so; fi
  for c in 5 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-sustained --no-same-level > gpurun_out/o_${c}_$tag.json 2>/dev/null
  echo "c$c $tag: $(python tools/bench_brief.py gpurun_out/o_${c}_$tag.json | grep -E "'role': 'restrict'" | sed -E "s/.*'ms': ([0-9.]+).*'frac_hbm': ([0-9.]+).*/\1ms \2/" | tr '\n' ' ') $(python tools/bench_brief.py gpurun_out/o_${c}_$tag.json | grep -o "'sm_mhz': [0-9.]*")"
  done
done; done
