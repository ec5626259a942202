# one iteration: GPU tests (optional, TESTS=1), benches of CFGS, k_ingest phase profile (K4PROF=1)
O=gpurun_out/iter
rm -rf $O; mkdir -p $O
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; fi
for c in ${CFGS:-c4 c1}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_${c}.log 2>&1
done
if [ -n "$K4PROF" ]; then
  for c in c4 c3; do
    SS_B200_LIB=$PWD/paper_1309_0634_b200/_lib/libss_k4prof.so timeout 300 python scripts/k4_prof.py --config $c > $O/k4prof_$c.log 2>&1
  done
fi
echo done
