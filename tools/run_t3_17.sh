# tile3 at p = 17 (TH_TILE3=2) vs the per-warp slide (TH_TILE3=1 = one-tile faces only), config 4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "alternative_kernel_paths" 2>&1 | tail -3
TH_TILE3=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "interp" 2>&1 | tail -3
for v in 2 1 2 1; do
  TH_TILE3=$v timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --cpu-sample 16 > gpurun_out/t3_c4_$v.json 2> gpurun_out/t3_c4_$v.err
  python tools/passes.py tile3=$v < gpurun_out/t3_c4_$v.json
done
