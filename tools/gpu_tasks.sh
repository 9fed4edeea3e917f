#!/bin/bash
# One parameterised driver for gpurun calls (replaces the round-1 one-off scripts):
#   gpurun -- 'bash tools/gpu_tasks.sh <task> [<task> ...]'
# Tasks write into gpurun_out/.  Each step has its own timeout so a hung kernel cannot
# hold the box.
mkdir -p gpurun_out
for task in "$@"; do
  echo "== $task"
  case "$task" in
    tests)      timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 ;;
    multi)      timeout 600 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -x 2>&1 | tail -5 ;;
    smoke)      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
    bench)      timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
                python tools/bench_brief.py gpurun_out/bench.json ;;
    bench_fast) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err; tail -3 gpurun_out/bench_fast.err
                python tools/bench_brief.py gpurun_out/bench_fast.json ;;
    ref)        timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -c 600 gpurun_out/ref.json ;;
    c[1-4])     n=${task#c}; timeout 900 python bench.py --config $n --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_c$n.json 2> gpurun_out/bench_c$n.err; tail -3 gpurun_out/bench_c$n.err
                python tools/bench_brief.py gpurun_out/bench_c$n.json ;;
    torchrun2)  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; tail -c 400 gpurun_out/torchrun1.json ;;
    *)          echo "unknown task $task" ;;
  esac
done
