set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
for c in c2 c1 c3 c2split c4; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
done
echo done
