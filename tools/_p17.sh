TH_TILE3=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "order3 or pool_interp" 2>&1 | tail -1
for v in 1 2 1 2; do TH_TILE3=$v timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-same-level > gpurun_out/p17_$v.json 2>/dev/null; echo "c4 tile3=$v"; python tools/bench_brief.py gpurun_out/p17_$v.json | sed -n 3,6p; done
