# Round evidence: gpu tests, smoke, full default bench (with cpu_baseline), reference arm,
# ncu launch list of the bench command.  Run under gpurun; outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
tail -5 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^E   " gpurun_out/pytest_gpu.log | head -20; tail -3 gpurun_out/smoke.log
tail -c 2500 gpurun_out/bench_full.log; tail -c 1200 gpurun_out/bench_ref.log
