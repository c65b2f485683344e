# Per-launch DRAM traffic of the frame kernels (one C2 frame, every launch of
# each kernel, ncu --set full) -> profiles/ncu_traffic.json via
# scripts/ncu_traffic.py.  Run under gpurun; raw reports in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-traffic}
for k in k_mlp_tc:6:6 k_march:7:7 k_place:6:6; do  # launches per C2 frame with grouped rounds (G=2)
  IFS=: read name skip count <<< "$k"
  timeout 900 ncu --set full --clock-control none -k regex:$name -s $skip -c $count \
    -o gpurun_out/${TAG}_$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 \
    > gpurun_out/${TAG}_$name.log 2>&1
  echo "$name rc=$?"
done
python scripts/ncu_traffic.py --workload c2 gpurun_out/${TAG}_k_mlp_tc.ncu-rep gpurun_out/${TAG}_k_march.ncu-rep \
  gpurun_out/${TAG}_k_place.ncu-rep > gpurun_out/ncu_traffic.json
cat gpurun_out/ncu_traffic.json
