set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "int64" > gpurun_out/gpu_tests_int64.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 300 -c 3 -o gpurun_out/prof_ingest_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 200 -c 2 -o gpurun_out/prof_sort_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 100 -c 1 -o gpurun_out/prof_sort_c1 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count -s 6 -c 1 -o gpurun_out/prof_count_c2 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu4.log 2>&1
echo done
