set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
for c in c4 c4u c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py > $O/memcheck.log 2>&1
echo done
