# tile_interp: L2 prefetch of the tile after next (TH_PREFETCH bit 16) A/B, config 2 and config 1
TH_PREFETCH=25 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "interp" 2>&1 | tail -2
for v in 25 9 25 9; do
  TH_PREFETCH=$v timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/tpf_c2_$v.json 2> gpurun_out/tpf_c2_$v.err
  python tools/passes.py c2pf=$v < gpurun_out/tpf_c2_$v.json
  TH_PREFETCH=$v timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/tpf_c1_$v.json 2> gpurun_out/tpf_c1_$v.err
  python tools/passes.py c1pf=$v < gpurun_out/tpf_c1_$v.json
done
