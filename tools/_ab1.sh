for sc in 0.125 1.0 0.125; do
timeout 600 python bench.py --scale $sc --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/sc_$sc.json 2> gpurun_out/sc_$sc.err
echo "scale $sc"; python tools/bench_brief.py gpurun_out/sc_$sc.json | head -4
done
