# Round-2 check: gpu tests, smoke, default bench, short reference arm.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
nproc > gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rA ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
if [ -n "$REF" ]; then timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-2} --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log; fi
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu.log | head -20; grep "C2 " gpurun_out/pytest_gpu.log | head -20; tail -3 gpurun_out/smoke.log
tail -c 1500 gpurun_out/bench_full.log; tail -c 800 gpurun_out/bench_ref.log 2>/dev/null
