# round 2: K4 shared share round, syncwarp fix; hash block A/B; tests
set -x
O=gpurun_out/r2l
mkdir -p $O
L=paper_1309_0634_b200/_lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static -diag-suppress 177,550 -DSS_K4_PROF paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_k4prof.so > $O/b1.log 2>&1
for c in c4 c5 c3; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
for b in 16 32; do
  SS_B200_HASH_BLOCK=$b timeout 400 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $O/bench_c4_blk$b.log 2>&1
  SS_B200_HASH_BLOCK=$b timeout 400 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu > $O/bench_c5_blk$b.log 2>&1
done
SS_B200_LIB=$L/libss_b200_k4prof.so SS_PROF_FN=ss_debug_k4_prof timeout 300 python scripts/sort_phase_prof.py c4 > $O/k4prof_c4.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
echo done
