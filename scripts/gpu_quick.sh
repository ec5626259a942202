set -x
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
for c in c2 c1 c3 c2split c4; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python bench.py --config c2 --initial contiguous --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2_contig.log 2>&1
echo done
