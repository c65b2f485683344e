# ncu --set full of N consecutive launches of one kernel inside the C2 bench:
#   KERNEL=k_mlp_tc SKIP=12 COUNT=6 NAME=r02b_mlp bash scripts/gpu_prof_one.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -s ${SKIP:-12} -c ${COUNT:-6} \
  -o gpurun_out/prof_${NAME} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_${NAME}.log 2>&1
echo "ncu rc=$?"
