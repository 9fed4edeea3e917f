mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_same_level.py -q -m gpu 2>&1 | tail -2
for c in 2 4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sl_c$c.json 2> gpurun_out/sl_c$c.err || tail -20 gpurun_out/sl_c$c.err
python -c "import json; d=json.load(open('gpurun_out/sl_c$c.json')); print($c, d['same_level'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/r1_prof_same_level3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_sl.log 2>&1; tail -1 gpurun_out/ncu_sl.log
