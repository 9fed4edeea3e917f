for c in 16 32 64; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 3 --e2e-chunks $c > gpurun_out/e2e_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); e=d['e2e']; print('chunks $c', round(e['value']/1e9,3), 'G/s', e['ms_per_step'], 'ms', e['matches_device_run'])"
done
