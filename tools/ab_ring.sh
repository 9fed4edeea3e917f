#!/bin/bash
# A/B of the slice-ring interpolation kernel (TH_RING) against the defaults:
#   gpurun -- 'bash tools/ab_ring.sh parity|bench [NA ...]'   (TH_RING=15: the ring for every interpolation)
mkdir -p gpurun_out
mode=$1; shift
sel="exchange_all_faces_small or pool_interp_batch or pool_interp_long_batch or pool_restrict_batch or transposed or unknown_counts"
if [ "$mode" = parity ]; then
  for na in "$@"; do
    echo "== parity TH_RING=15 NA=$na"
    TH_RING=15 TH_RING_NA=$na timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "$sel" 2>&1 | tail -4
  done
else
  for cfg in 3 4; do
    echo "== config $cfg default"
    timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-same-level > gpurun_out/ring_c${cfg}_def.json 2> gpurun_out/ring_c${cfg}_def.err
    python tools/bench_brief.py gpurun_out/ring_c${cfg}_def.json | grep -E "interpolate|parity"
    for na in "$@"; do
      echo "== config $cfg TH_RING=15 NA=$na"
      TH_RING=15 TH_RING_NA=$na timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-same-level > gpurun_out/ring_c${cfg}_na$na.json 2> gpurun_out/ring_c${cfg}_na$na.err
      tail -2 gpurun_out/ring_c${cfg}_na$na.err
      python tools/bench_brief.py gpurun_out/ring_c${cfg}_na$na.json | grep -E "interpolate|parity"
    done
  done
fi
