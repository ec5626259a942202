# round-2 starting point: C4/C3/C5 launch lists and benches
set -x
O=gpurun_out/r2base
mkdir -p $O
for c in c4 c3 c4u; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for c in c4 c4u; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
echo done
