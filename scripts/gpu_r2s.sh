# round 2: pipelined int64 key probe: tests, benches with / without
set -x
O=gpurun_out/r2s
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "int64" > $O/int64_tests.log 2>&1
for c in c4 c5 c4u; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
  SS_B200_NO_KEY_PIPE=1 timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_${c}_nopipe.log 2>&1
done
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
echo done
