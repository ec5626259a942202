# timing ablations of the placement kernel (results are wrong by design)
O=gpurun_out/abl; mkdir -p $O
for v in "" $ABL; do
  if [ -z "$v" ]; then L=paper_1309_0634_b200/_lib/libss_b200.so; else L=paper_1309_0634_b200/_lib/libss_b200_abl$v.so; fi
  SS_B200_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sort_pass -c 40 --csv --log-file $O/sort$v.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
echo done
