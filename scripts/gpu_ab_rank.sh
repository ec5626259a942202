# A/B of the single-pass placement (k_rank_place) against the radix passes
set -x
O=gpurun_out/abrank
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
for c in ${CFGS:-c1 c2 c2split}; do
  for r in 0 1; do
    SS_B200_RANK_PLACE=$r timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_${c}_r$r.log 2>&1
  done
done
echo done
