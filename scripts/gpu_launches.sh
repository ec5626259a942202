# per-kernel launch lists (serialised, cold-cache) for every config + default bench
set -x
O=gpurun_out/launch
mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 5 --cpu-seconds 10 > $O/bench_default.log 2>&1
for c in c1 c2 c3 c4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu_$c.log 2>&1
done
echo done
