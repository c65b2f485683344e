# Full evidence pass for profiles/: tests, smoke, default bench (with
# cpu_baseline), reference arm, c4/c5 legs, launch list, ncu --set full of the
# three frame kernels at a heavy round, per-launch DRAM traffic.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-final}
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1
for k in k_mlp_tc:${MLP_SKIP:-8} k_march:${MARCH_SKIP:-9} k_place:${PLACE_SKIP:-8} k_ray_init:1 k_extract_analytic:1 k_grouped_backward:2 k_bwd_tc:2 k_photo_ray:2; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o gpurun_out/prof_${TAG}_$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1
done
TAG=traffic bash scripts/gpu_traffic.sh > /dev/null 2>&1
rm -f gpurun_out/traffic_*.ncu-rep   # large multi-launch captures: only their JSON summary travels back
du -sh gpurun_out
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; ls gpurun_out | head -50
