# k_rank_place matching mix: of every 4 rounds, b by ballots (rest MATCH)
O=gpurun_out/rankvar
rm -rf $O; mkdir -p $O
timeout 300 python bench.py --config c2split --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_b2.log 2>&1
for b in 1 3; do
  SS_B200_LIB=$PWD/paper_1309_0634_b200/_lib/var_b$b.so timeout 300 python bench.py --config c2split --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_b$b.log 2>&1
done
