set -x
O=gpurun_out/os2
mkdir -p $O
python scratch/dbg_os.py > $O/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_placement.py -q -x > $O/tests.log 2>&1
for c in c4 c3 c5 c4u; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
echo done
