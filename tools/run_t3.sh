# order3 tile interpolation A/B on one B200 (run from the repo root under gpurun)
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
for v in 1 0 1 0; do
  TH_TILE3=$v timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --cpu-sample 16 > gpurun_out/t3_c3_$v.json 2> gpurun_out/t3_c3_$v.err
  python tools/passes.py tile3=$v < gpurun_out/t3_c3_$v.json
done
if [ -n "$T3_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile3" -s 1 -c 1 -o gpurun_out/t3_prof python bench.py --config 3 --scale 0.25 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/t3p_ncu.log 2>&1
tail -1 gpurun_out/t3p_ncu.log
fi
