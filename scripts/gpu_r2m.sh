# round 2: split planned on values to store; tests, benches, C3 policy comparison
set -x
O=gpurun_out/${R2TAG:-r2m}
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
for c in c3 c4 c5 c2 c1; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 900 python scripts/compare_policies.py --config c3 --steps 6 --warmup 12 > $O/compare_c3.log 2>&1
echo done
