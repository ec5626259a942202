set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config c2split --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2split.log 2>&1
echo done
