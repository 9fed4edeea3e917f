# tile3 diagnosis: failing test detail + ncu of the order3 tile kernel (config 3 at scale 0.25)
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k functional_api 2>&1 | grep -v "^\s*$" | tail -40
timeout 300 python bench.py --config 3 --scale 0.25 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/t3p_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile3" -s 1 -c 1 -o gpurun_out/t3_prof python bench.py --config 3 --scale 0.25 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/t3p_ncu.log 2>&1
tail -3 gpurun_out/t3p_ncu.log
