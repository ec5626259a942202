# quick status pass: smoke, GPU tests, every bench config (no CPU leg)
set -x
O=gpurun_out/status
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_default.log 2>&1
for c in c1 c3 c4 c2split; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1
echo done
