# quick check: GPU tests + short benches of every config (+ optional launch lists)
set -x
O=gpurun_out/quick
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
for c in c1 c2 c2split c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for c in $LAUNCH_CFGS; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
echo done
