cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for v in "GF_NO_COARSE=1" "GF_COARSE_FACTOR=1" "GF_COARSE_FACTOR=2" "GF_COARSE_FACTOR=4"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
s=d['stage_roofline']; print('$v', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_frame'],3), {k:round(v['ms_per_frame'],3) for k,v in s.items()}, 'Q', d['queries_per_frame'])"
done
