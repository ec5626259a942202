# round 2: int64-key sharding tests + the full GPU suite
set -x
O=gpurun_out/r2o
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > $O/sharded.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
timeout 400 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > $O/bench_c1.log 2>&1
echo done
