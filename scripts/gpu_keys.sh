set -x
O=gpurun_out/keys
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -k "int64 or keys or c4 or C4 or fullsize" > $O/tests.log 2>&1
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
