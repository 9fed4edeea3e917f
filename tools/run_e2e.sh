# e2e pipeline depth A/B (config 2, through the C ABI with host buffers)
for c in 8 16 32 8 16 32; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 3 --e2e-chunks $c > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err
  python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); e=d['e2e']; print('chunks $c', round(e['value']/1e9,3), 'G/s', e['ms_per_step'], 'ms', e['matches_device_run'])"
done
