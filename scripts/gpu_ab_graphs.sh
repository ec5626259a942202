# A/B: CUDA graphs on/off for every config
set -x
O=gpurun_out/ab; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
for c in c1 c2 c2split c3 c4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu > $O/bench_$c.log 2>&1
  SS_B200_NO_GRAPHS=1 timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu > $O/bench_${c}_nog.log 2>&1
done
echo done
