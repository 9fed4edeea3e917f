# tile3 CTA shape A/B: TH_TILE3_CFG=1 (chunks of 20, 192 threads x 3 CTAs/SM, flattened items)
# (TH_TILE3_CFG was removed after this A/B: profiles/r01_ab_tile3.txt)
# vs 0 (chunks of 31, 288 x 2, warp-aligned; default)
TH_TILE3_CFG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "interp" 2>&1 | tail -2
for v in 1 0 1 0; do
  TH_TILE3_CFG=$v timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --cpu-sample 16 > gpurun_out/t3cfg_$v.json 2> gpurun_out/t3cfg_$v.err
  python tools/passes.py cfg=$v < gpurun_out/t3cfg_$v.json
done
