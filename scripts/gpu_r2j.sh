# round 2: chain-free small-G placement (k_rank_small), key count default, tests
set -x
O=gpurun_out/r2j
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
for c in c1 c4 c2; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 30 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
