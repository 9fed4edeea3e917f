# p = 17 order2 / tensor interpolation: staged tiles in 3 x 3 spatial tiles (TH_TILE_MULTI=1, now
# with the L2 prefetch of the tile after next) vs the per-warp slide (default), config 4
for v in 1 0 1 0; do
  TH_TILE_MULTI=$v timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/m17_$v.json 2> gpurun_out/m17_$v.err
  python tools/passes.py multi=$v < gpurun_out/m17_$v.json
done
