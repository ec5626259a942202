# A/B of a variant library (VAR_LIB) against the built one on CFGS
O=gpurun_out/var
rm -rf $O; mkdir -p $O
for c in ${CFGS:-c2 c2split}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_${c}_base.log 2>&1
  SS_B200_LIB=$PWD/$VAR_LIB timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_${c}_var.log 2>&1
done
