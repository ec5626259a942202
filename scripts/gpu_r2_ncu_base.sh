# round-2 baseline ncu --set full captures at C4/C3 + all-policy comparison at C4
set -x
O=gpurun_out/r2ncu
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_key_probe|k_sort_pass|k_ingest|k_count|k_ring_copy|k_finalize|k_minmax_rescan|k_batch_stats' -s 40 -c 9 -o $O/full_c4 $B --config c4 > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sort_pass|k_ingest|k_count|k_batch_stats|k_finalize' -s 25 -c 6 -o $O/full_c3 $B --config c3 > $O/ncu_c3.log 2>&1
timeout 1500 python scripts/compare_policies.py --config c4 --steps 6 --warmup 3 > $O/compare_c4.log 2>&1
echo done
