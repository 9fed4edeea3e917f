# tile3w (TH_TILE3=3: one 18-warp CTA per SM, double-buffered box) vs tile3 (TH_TILE3=1)
# (the TH_TILE3=3 variant was removed after this A/B: profiles/r01_ab_tile3.txt)
TH_TILE3=3 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "interp" 2>&1 | tail -2
for v in 3 1 3 1; do
  TH_TILE3=$v timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --cpu-sample 16 > gpurun_out/t3w_$v.json 2> gpurun_out/t3w_$v.err
  python tools/passes.py tile3=$v < gpurun_out/t3w_$v.json
done
