# A/B: int64 key count at 2 vs 3 CTAs per SM (register budget)
set -x
O=gpurun_out/r2u
mkdir -p $O
L=paper_1309_0634_b200/_lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static -diag-suppress 177,550 -DSS_KEY_MINB=3 paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_k3.so > $O/b.log 2>&1
for c in c4 c4u; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
  SS_B200_LIB=$L/libss_b200_k3.so timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_${c}_k3.log 2>&1
done
echo done
