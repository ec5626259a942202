# full measurement pass: tests, smoke, headline bench (with CPU baseline),
# other configs, reference arm, launch lists + ncu --set full captures
set -x
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c2.log 2>&1
for c in c1 c2split c3 c4 c4u c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 400 python bench.py --config c1 --steps 10 --warmup 3 --cpu-seconds 10 > $O/bench_c1_cpu.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 --cpu-seconds 12 > $O/bench_ref.log 2>&1
for c in c1 c2 c3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_rank_place|k_ingest|k_count|k_batch_stats|k_balance" -s 25 -c 6 -o $O/full_c2 $B > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_ingest|k_count|k_batch_stats|k_scan|k_finalize|k_chunk" -s 21 -c 7 -o $O/full_c1 $B --config c1 > $O/ncu_c1.log 2>&1
echo done
