set -x
O=gpurun_out/bk2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_bucket.py tests/test_gpu_parity.py -q -x > $O/tests.log 2>&1
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
SS_B200_BUCKET=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bk_scatter|k_bk_local|k_bk_hist|k_key_count' -s 30 -c 4 -o $O/full_bk_c4 $B --config c4 > $O/ncu_c4.log 2>&1
echo done
