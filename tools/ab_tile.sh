# same-call A/B of the staged tile interpolation (TH_TILE=1, TH_TILE_CFG variants) vs the per-warp slide (TH_TILE=0)
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for cfg in "--config 2" "--config 1"; do
  for t in "TH_TILE_CFG=0" "TH_TILE_CFG=1" "TH_TILE_CFG=3" "TH_TILE_CFG=4" "TH_TILE=0"; do
    env $t timeout 300 python bench.py $cfg --steps 20 --warmup 3 --no-e2e --cpu-sample 16 2>/dev/null | python tools/passes.py "$t"
  done
done
