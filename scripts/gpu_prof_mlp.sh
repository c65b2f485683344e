cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 17 -c 1 \
  -o gpurun_out/prof_mlp_tc2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp2.log 2>&1
echo "mlp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march -s 19 -c 1 \
  -o gpurun_out/prof_march2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_march2.log 2>&1
echo "march rc=$?"
