# full measurement pass on one B200 (run from the repo root under gpurun)
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 600 python bench.py > gpurun_out/r1_c2.json 2> gpurun_out/r1_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-sample 64 > gpurun_out/r1_c$c.json 2> gpurun_out/r1_c$c.err; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"restrict_reg|gram_slide|tile_interp" -s 4 -c 4 -o gpurun_out/r1_prof_c2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_f.log 2>&1
timeout 300 python bench.py --config 3 --scale 0.25 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stage_slide|tile3" -c 2 -o gpurun_out/r1_prof_c3 python bench.py --config 3 --scale 0.25 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_f3.log 2>&1
tail -1 gpurun_out/ncu_f.log gpurun_out/ncu_f3.log
# the torchrun launch path (one rank; the driver's N > 1 runs use the same code path)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r1_torchrun1.json 2> gpurun_out/r1_torchrun1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r1_torchrun1_ref.json 2> gpurun_out/r1_torchrun1_ref.err
