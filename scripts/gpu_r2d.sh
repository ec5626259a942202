# round 2 (re-entry): smoke, GPU suite, headline bench (C4) + other configs,
# reference arm, C4 launch list, ncu --set full of the C4 kernels
set -x
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_default.log 2>&1
for c in c1 c2 c3 c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_key|k_sort|k_os_|k_lsd|k_ingest|k_count|k_ring_copy|k_finalize|k_minmax|k_batch_stats|k_tile' -s 40 -c 10 -o $O/full_c4 $B --config c4 > $O/ncu_c4.log 2>&1
echo done
