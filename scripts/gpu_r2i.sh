# round 2: block-hash partitions (8-id blocks), k_os_pass vector zeroing; A/B: contiguous map, 32-bit key hash, no key-count aggregation
set -x
O=gpurun_out/r2i
mkdir -p $O
L=paper_1309_0634_b200/_lib
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static -diag-suppress 177,550"
nvcc $F -DSS_KEY_HASH32 paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_h32.so > $O/b1.log 2>&1
for c in c4 c5 c3 c2 c1; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for c in c4 c5 c3; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --initial contiguous > $O/bench_${c}_contig.log 2>&1
done
SS_B200_LIB=$L/libss_b200_h32.so timeout 400 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4_h32.log 2>&1
SS_B200_KEY_AGG=0 timeout 400 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4_agg0.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
echo done
