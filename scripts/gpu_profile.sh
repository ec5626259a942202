set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 31 -c 1 -o gpurun_out/prof_ingest_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 28 -c 1 -o gpurun_out/prof_ingest_c2split python bench.py --config c2split --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu1b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rank_place -s 24 -c 1 -o gpurun_out/prof_rank_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 24 -c 1 -o gpurun_out/prof_sort_c1 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu3.log 2>&1
echo done
