# same-call A/B of the working tree's library against _lib_ab/base (tools/ab_build.sh <rev> base)
# usage: bash tools/ab_lib.sh "<bench args>" ["<bench args>" ...]
for cfg in "$@"; do
  for lib in new base; do
    if [ $lib = base ]; then export TH_LIBPATH=$PWD/_lib_ab/base/libtrihalo_b200.so; else unset TH_LIBPATH; fi
    timeout 300 python bench.py $cfg --steps 20 --warmup 3 --no-e2e --cpu-sample 16 2>/dev/null | python tools/passes.py "$lib"
  done
done
