# ncu --set full captures of the top kernels (steady state, after warm-up)
set -x
O=gpurun_out/full
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rank_place -s 3 -c 1 -o $O/rank_c2 $B > $O/l1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 3 -c 1 -o $O/ingest_c2 $B > $O/l2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_balance -s 3 -c 1 -o $O/balance_c2 $B > $O/l6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan_reduce|k_batch_stats|k_count|k_sort_pass|k_ingest|k_finalize' -s 18 -c 6 -o $O/small_c1 $B --config c1 > $O/l3.log 2>&1
echo done
