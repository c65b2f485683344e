cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for v in ${C5_VARIANTS:-GF_X=0}; do
  env $v timeout 300 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/b.log') if l.startswith('{')][-1]); s=d.get('stage_ms'); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in s.items()})"
done
