# A/B: interpolation passes on a side stream beside the restrictions (bench.py --overlap)
mkdir -p gpurun_out
for r in 1 2; do
  for c in 2 4 3; do
    for o in "" "--overlap"; do
      st=50; [ $c != 2 ] && st=10
      timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu $o > gpurun_out/ov.json 2>gpurun_out/ov.err || tail -5 gpurun_out/ov.err
      python -c "import json; d=json.load(open('gpurun_out/ov.json')); print('c$c', 'overlap' if '$o' else 'serial ', round(d['value']/1e9,2), 'G/s', round(d['ms_per_step'],3), 'ms/step', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
