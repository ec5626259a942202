set -x
O=gpurun_out/os
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_fullsize.py -q -x -k "not bucket-1 and not -1-" > $O/tests.log 2>&1
for c in c4 c3 c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_os_pass|k_os_up' -s 40 -c 3 -o $O/full_os_c4 $B --config c4 > $O/ncu_c4.log 2>&1
echo done
