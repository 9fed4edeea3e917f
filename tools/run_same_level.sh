# same-level halo fill: parity tests + bench legs (configs 2, 4) + one ncu --set full capture of the copy kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_same_level.py tests/test_capi.py -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/sl_c2.json 2> gpurun_out/sl_c2.err || tail -20 gpurun_out/sl_c2.err
python -c "import json; d=json.load(open('gpurun_out/sl_c2.json')); print(d['value']/1e9, d['same_level'])"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sl_c4.json 2> gpurun_out/sl_c4.err || tail -20 gpurun_out/sl_c4.err
python -c "import json; d=json.load(open('gpurun_out/sl_c4.json')); print(d['value']/1e9, d['same_level'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/r1_prof_same_level python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_sl.log 2>&1; tail -2 gpurun_out/ncu_sl.log
