# MLP kernel iteration: smoke (hang guard), fp16 parity tests, bench A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
GF_DEBUG=1 timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -4 gpurun_out/smoke.log
if grep -q "smoke rc=0" gpurun_out/smoke.log; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^E   " gpurun_out/pytest_gpu.log | head -20
  for v in ${GF_AB_VARIANTS:-"GF_X=0"}; do
    env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab.log 2>&1 || tail -5 gpurun_out/bench_ab.log
    python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
s=d['stage_roofline']; print('$v', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_frame'],3), {k:round(v['ms_per_frame'],3) for k,v in s.items() if isinstance(v, dict)}, 'Q', d['queries_per_frame'], 'clk', d['clocks']['sm_mhz'])"
  done
fi
