# round 2: C1 count-chunk size A/B
set -x
O=gpurun_out/r2r
mkdir -p $O
for sb in 65536 32768 131072; do
  timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu --sub-batch $sb > $O/bench_c1_$sb.log 2>&1
done
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --sub-batch 32768 > $O/bench_c2_32768.log 2>&1
echo done
