cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 12 -c 6 \
  -o gpurun_out/prof_r02_mlp_tc -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_r02_mlp.log 2>&1
echo "mlp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march -s 14 -c 7 \
  -o gpurun_out/prof_r02_march -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_r02_march.log 2>&1
echo "march rc=$?"
