cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1; echo "launches rc=$?"
for k in k_march:20 k_scatter_render:17 k_scan_cells:17 k_ray_init:1; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o gpurun_out/prof_$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1
  echo "$name rc=$?"
done
