for v in random siblings random siblings; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --fine-layout $v > gpurun_out/lay_$v.json 2>/dev/null; echo "c5 $v"; python tools/bench_brief.py gpurun_out/lay_$v.json | sed -n 1,4p
done
