set -x
O=gpurun_out/bucket
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bucket.py -q -x > $O/tests.log 2>&1
for c in c4 c3 c4u c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
