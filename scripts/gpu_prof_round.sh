# ncu --set full captures of the four frame kernels at a heavy round of the
# second C2 frame (bench command, one GPU).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-v5}
for k in ${KERNELS:-k_mlp_tc:17 k_march:18 k_place:17 k_ray_init:1}; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o gpurun_out/prof_${TAG}_$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 \
    > gpurun_out/prof_${TAG}_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out | grep prof_
