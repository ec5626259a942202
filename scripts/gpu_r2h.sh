# round 2: K4 thread-contiguous short path A/B, k_os_pass phase profile, tests
set -x
O=gpurun_out/r2h
mkdir -p $O
L=paper_1309_0634_b200/_lib
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static -diag-suppress 177,550"
nvcc $F -DSS_K4_SHORT_LANES paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_oldshort.so > $O/b1.log 2>&1
nvcc $F -DSS_SORT_PROF paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_sortprof.so > $O/b2.log 2>&1
nvcc $F -DSS_K4_PROF paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_k4prof.so > $O/b3.log 2>&1
for c in c4 c2 c1 c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
  SS_B200_LIB=$L/libss_b200_oldshort.so timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_${c}_old.log 2>&1
done
SS_B200_LIB=$L/libss_b200_sortprof.so SS_PROF_OS=1 timeout 300 python scripts/sort_phase_prof.py c4 > $O/osprof_c4.log 2>&1
SS_B200_LIB=$L/libss_b200_k4prof.so SS_PROF_FN=ss_debug_k4_prof timeout 300 python scripts/sort_phase_prof.py c4 > $O/k4prof_c4.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
echo done
