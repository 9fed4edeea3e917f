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
    ncu_c5)     # launch list of the default bench (config 5) + one full-set capture of both kernels (config 5 at 1/8 scale)
                cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
                timeout 600 $cmd > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err &&
                timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tile3|stage_slide|strided_box|finite" -c 40 --csv --log-file gpurun_out/launches_c5.csv $cmd > gpurun_out/ncu_list.log 2>&1
                cmd8="python bench.py --scale 0.125 --steps 1 --warmup 1 --no-e2e --no-cpu"
                timeout 600 $cmd8 > gpurun_out/ncu_plain8.json 2>&1 &&
                timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tile3p|stage_slide" -s 2 -c 2 -o gpurun_out/prof_c5 -f $cmd8 > gpurun_out/ncu_full.log 2>&1
                tail -2 gpurun_out/ncu_full.log ;;
    ncu_cfg[1-4]) # launch list + one full-set capture of every interpolation / restriction kernel of config N
                n=${task#ncu_cfg}; cmd="python bench.py --config $n --steps 1 --warmup 1 --no-e2e --no-cpu --no-same-level"
                timeout 600 $cmd > gpurun_out/ncu_plain_c$n.json 2> gpurun_out/ncu_plain_c$n.err &&
                timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"ring_interp|tile3p|tile_interp|stage_slide|restrict_reg|gram_slide" -s $(( n == 3 ? 4 : 8 )) -c 4 -o gpurun_out/prof_c$n -f $cmd > gpurun_out/ncu_full_c$n.log 2>&1
                tail -2 gpurun_out/ncu_full_c$n.log ;;
    reftests)   # the reference's own tests against the drop-in (needs baseline/_ref/tests_ref, git-ignored)
                timeout 1200 python tools/run_reference_tests.py baseline/_ref/tests_ref test_schemes.py -q > gpurun_out/reftests_schemes.log 2>&1; tail -3 gpurun_out/reftests_schemes.log
                timeout 1800 python tools/run_reference_tests.py baseline/_ref/tests_ref test_acceptance.py -q -k "criterion_1 or criterion_2 or criterion_3 or criterion_4" > gpurun_out/reftests_acceptance.log 2>&1; tail -3 gpurun_out/reftests_acceptance.log
                timeout 1800 python tools/run_reference_tests.py baseline/_ref/tests_ref -q -rf --ignore=baseline/_ref/tests_ref/test_cli.py > gpurun_out/reftests_all.log 2>&1; grep -E "^FAILED|passed|failed" gpurun_out/reftests_all.log | tail -30 ;;
    latency)    timeout 1200 python tools/per_face_latency.py > gpurun_out/per_face_latency.json 2> gpurun_out/per_face_latency.err; tail -12 gpurun_out/per_face_latency.err ;;
    refcpu)     timeout 1200 python tools/reference_cpu.py 256 > gpurun_out/reference_cpu.json 2> gpurun_out/reference_cpu.err; cat gpurun_out/reference_cpu.json ;;
    matrix)     timeout 900 python bench.py --config 2 --passes interpolate:matrix_linear,restrict:matrix_linear,interpolate:tensor_linear,restrict:tensor_linear --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_matrix.json 2> gpurun_out/bench_matrix.err; tail -3 gpurun_out/bench_matrix.err
                python tools/bench_brief.py gpurun_out/bench_matrix.json ;;
    *)          echo "unknown task $task" ;;
  esac
done
