# one ncu --set full capture: $1 = kernel regex, $2 = skip, $3 = count, $4 = name, rest = bench args
set -x
O=gpurun_out/full
mkdir -p $O
K=$1; S=$2; C=$3; N=$4; shift 4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $C -o $O/$N python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 "$@" > $O/$N.log 2>&1
echo done
