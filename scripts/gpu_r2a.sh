# round-2 first GPU pass: tests, smoke, default bench (C4), other configs, launch lists
set -x
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
nproc > $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_default.log 2>&1
for c in c1 c2 c3 c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for c in c4 c3 c2; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
echo done
