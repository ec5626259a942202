# round 2: key-count fast path, per-group grids; all-policy comparison at C4 and C3
set -x
O=gpurun_out/r2k
mkdir -p $O
for c in c4 c5 c3 c1; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 40 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 1500 python scripts/compare_policies.py --config c4 --steps 6 --warmup 12 > $O/compare_c4.log 2>&1
timeout 900 python scripts/compare_policies.py --config c3 --steps 6 --warmup 12 > $O/compare_c3.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
echo done
