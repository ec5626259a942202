set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 200 python scripts/diag_k4.py c2 > gpurun_out/diag_c2.log 2>&1
timeout 200 python scripts/diag_k4.py c2split > gpurun_out/diag_c2split.log 2>&1
for c in c2 c1 c3 c2split; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
done
echo done
