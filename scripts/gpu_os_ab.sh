# A/B: onesweep digit width x match mode, and the CTA-wide balancer at C4
set -x
O=gpurun_out/osab
mkdir -p $O
for c in c4 c4u c3; do
  for b in 7 10; do
    for m in 0 1 2; do
      SS_B200_OS_BITS=$b SS_B200_OS_MATCH=$m timeout 300 python bench.py --config $c --steps 8 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_${c}_b${b}_m${m}.log 2>&1
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k movelists > $O/tests_mv.log 2>&1
timeout 1500 python scripts/compare_policies.py --config c4 --steps 6 --warmup 3 > $O/compare_c4.log 2>&1
echo done
