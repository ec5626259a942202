set -x
O=gpurun_out/r2t
mkdir -p $O
for c in c4 c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
  SS_B200_OS2=1 timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_${c}_os2.log 2>&1
done
SS_B200_OS2=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "int64 or c4 or C4" > $O/tests_os2.log 2>&1
echo done
