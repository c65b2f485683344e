# ncu evidence for the bench's C2 frame: launch list (cold, serialised) and
# full captures of the top kernels.  Run under gpurun; outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 29 -c 2 \
  -o gpurun_out/prof_mlp_tc -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp.log 2>&1
echo "mlp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march -s 31 -c 2 \
  -o gpurun_out/prof_march -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_march.log 2>&1
echo "march rc=$?"
ls -la gpurun_out
