# K4 work-proportional grid: total CTAs (x148) and static-partition use
O=gpurun_out/k4grid
rm -rf $O; mkdir -p $O
for wv in 2 4 8 16; do
  SS_B200_K4_WAVES=$wv timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_c2_w$wv.log 2>&1
done
for st in 0 1; do
  SS_B200_K4_STATIC=$st timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $O/bench_c1_s$st.log 2>&1
done
