mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in 2 4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sl_c$c.json 2> gpurun_out/sl_c$c.err || tail -20 gpurun_out/sl_c$c.err
python -c "import json; d=json.load(open('gpurun_out/sl_c$c.json')); print($c, d['same_level'])"
done
