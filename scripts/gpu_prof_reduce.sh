cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_reduce" -s 4 -c 1 \
  -o gpurun_out/prof_red -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1; echo "ncu rc=$?"
