# tile_interp small-batch unknown split (TH_TILE_SPLIT) A/B, config 1; parity of the split path
# (TH_TILE_SPLIT was removed after this A/B: profiles/r01_ab_tile.txt)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "interp or exchange_all" 2>&1 | tail -2
for v in 1 0 1 0; do
  TH_TILE_SPLIT=$v timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-e2e --cpu-sample 16 > gpurun_out/split_$v.json 2> gpurun_out/split_$v.err
  python tools/passes.py c1split=$v < gpurun_out/split_$v.json
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu | python tools/passes.py c2
