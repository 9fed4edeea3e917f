set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 600 python bench.py > gpurun_out/v_c2.json 2> gpurun_out/v_c2.err; cat gpurun_out/v_c2.json | head -c 600
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --cpu-sample 64 > gpurun_out/v_c4.json 2> gpurun_out/v_c4.err
