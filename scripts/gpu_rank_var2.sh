# k_rank_place ablations (timing only; VAR 1..4 drop the chain / stores / matching / atomics)
O=gpurun_out/rankabl
rm -rf $O; mkdir -p $O
timeout 300 python bench.py --config c2split --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_v0.log 2>&1
for v in 1 2 3 4; do
  SS_B200_LIB=$PWD/paper_1309_0634_b200/_lib/var_v$v.so timeout 300 python bench.py --config c2split --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_v$v.log 2>&1
done
