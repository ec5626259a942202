# round 2: K4 short-path register caching, key-mark grid; benches + K4 phases
set -x
O=gpurun_out/r2q
mkdir -p $O
L=paper_1309_0634_b200/_lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static -diag-suppress 177,550 -DSS_K4_PROF paper_1309_0634_b200/csrc/engine.cu -o $L/libss_b200_k4prof.so > $O/b1.log 2>&1
for c in c4 c5 c3 c2; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
SS_B200_LIB=$L/libss_b200_k4prof.so SS_PROF_FN=ss_debug_k4_prof timeout 300 python scripts/sort_phase_prof.py c4 > $O/k4prof_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 40 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
echo done
