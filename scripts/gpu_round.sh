# full measurement pass: tests, headline bench (with CPU baseline), other
# configs, reference arm, launch list + ncu captures of the top kernels
set -x
mkdir -p gpurun_out/round
O=gpurun_out/round
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c2.log 2>&1
for c in c1 c3 c4 c2split; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 12 > $O/bench_ref.log 2>&1
timeout 600 python scripts/compare_policies.py --config c2 --steps 4 --warmup 3 > $O/policies_c2.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 124 -c 4 -o $O/prof_ingest_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 48 -c 2 -o $O/prof_sort_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu2.log 2>&1
echo done
