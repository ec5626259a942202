# round-2 final measurement pass on the final code (three calls: gpurun copies back <= 64 MiB):
#   bash scripts/gpu_r2f.sh bench   smoke, headline bench (C4, with CPU baseline), other configs,
#                                   reference arm, steady-state launch lists C1-C5
#   bash scripts/gpu_r2f.sh ncu     ncu --set full of the top kernels, C4 and C1
#   bash scripts/gpu_r2f.sh extra   compute-sanitizer, all-policy comparison at C4 and C3
set -x
O=gpurun_out/r2f
mkdir -p $O
B="python bench.py --steps 30 --warmup 3 --no-cpu --e2e-steps 1"
case "$1" in
bench)
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
  nproc > $O/nproc.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  timeout 900 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
  timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.log 2>&1
  for c in c1 c2 c3 c4u c5; do
    timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
  done
  timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
  for c in c1 c2 c3; do
    timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 300 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 40 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  done
  for c in c4 c5; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 400 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 40 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  done
  ;;
ncu)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_key_count|k_os_pass|k_ingest|k_finalize|k_os_up|k_batch_stats' -s 120 -c 7 -o $O/full_c4 $B --config c4 > $O/ncu_c4.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_count_rows|k_rank_place|k_ingest|k_batch_stats|k_finalize|k_sub' -s 120 -c 6 -o $O/full_c1 $B --config c1 > $O/ncu_c1.log 2>&1
  ;;
extra)
  for c in c1 c2 c3 c4 c5; do
    timeout 300 python scripts/partition_times.py $c 12 > $O/parttimes_$c.log 2>&1
  done
  timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py > $O/memcheck.log 2>&1
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_cases.py > $O/racecheck.log 2>&1
  timeout 1500 python scripts/compare_policies.py --config c4 --steps 6 --warmup 12 > $O/compare_c4.log 2>&1
  timeout 900 python scripts/compare_policies.py --config c3 --steps 6 --warmup 12 > $O/compare_c3.log 2>&1
  ;;
esac
echo done
