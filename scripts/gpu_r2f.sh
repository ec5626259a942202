# round 2: device-resident multi-GPU plane, hot-key shared table, column-scan blocks
set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > $O/bench_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 30 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
