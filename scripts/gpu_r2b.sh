# round 2: full GPU suite + benches after the placement / balancer / pull changes
set -x
O=gpurun_out/r2b
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_default.log 2>&1
for c in c1 c2 c3 c4u c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for m in 0 1; do SS_B200_KEY_AGG=$m timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4_agg$m.log 2>&1; done
timeout 1500 python scripts/compare_policies.py --config c4 --steps 6 --warmup 3 > $O/compare_c4.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
