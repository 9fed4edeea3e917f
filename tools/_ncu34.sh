for c in 3 4; do
  cmd="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-same-level"
  timeout 600 $cmd > gpurun_out/ncu34_plain_$c.json 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile3p|gram_slide|tile_interp|stage_slide|restrict_reg" -s 4 -c 4 -f -o gpurun_out/prof_c$c $cmd > gpurun_out/ncu34_$c.log 2>&1
  tail -1 gpurun_out/ncu34_$c.log
done
