#!/bin/bash
# same-call A/B of library variants (_lib_ab/<tag>) with the slice ring on:
#   bash tools/ab_ring2.sh "<configs>" "<NA list>" tag1 tag2 ...   (tag "tree" = the in-tree library)
mkdir -p gpurun_out
cfgs=$1; nas=$2; shift 2
for cfg in $cfgs; do
  for tag in "$@"; do
    if [ $tag = tree ]; then unset TH_LIBPATH; else export TH_LIBPATH=$PWD/_lib_ab/$tag/libtrihalo_b200.so; fi
    for na in $nas; do
      out=gpurun_out/ring2_c${cfg}_${tag}_na$na
      TH_RING=${TH_RING_BITS:-15} TH_RING_NA=$na timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --cpu-sample 256 --no-same-level $BENCH_EXTRA > $out.json 2> $out.err
      echo "c$cfg $tag NA=$na: $(python tools/bench_brief.py $out.json | grep -E "interpolate" | sed -E "s/.*'scheme': '([a-z0-9_]+)'.*'ms': ([0-9.]+).*'frac_hbm': ([0-9.]+).*/\1 \2ms \3/" | tr '\n' ' ') $(python -c "import json,sys; d=json.loads(open('$out.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('parity', p.get('ok'), p.get('max_rel_err'))" 2>/dev/null || tail -1 $out.err | cut -c1-100)"
    done
  done
done
