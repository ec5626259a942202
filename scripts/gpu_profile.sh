set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_ingest -s 40 -c 1 -o gpurun_out/prof_ingest python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 60 -c 2 -o gpurun_out/prof_sort python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_count -s 6 -c 1 -o gpurun_out/prof_count python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu3.log 2>&1
echo done
