# GPU tests + short benches of the given configs (CFGS)
O=gpurun_out/check
rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
for c in ${CFGS:-c1 c2 c2split}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_${c}.log 2>&1
done
