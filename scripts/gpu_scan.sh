cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "configs or parity or query or group" > gpurun_out/pt_scan.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_scan.log; grep -E "^FAILED|^E  " gpurun_out/pt_scan.log | head
for w in c4 c5; do for v in GF_X=0 GF_SCAN_ONE_CTA=1; do
  env $v timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/b.log') if l.startswith('{')][-1]); s=d.get('stage_roofline') or d.get('stage_ms'); print('$w $v', round(d['ms_per_step'],3), {k:(round(v['ms_per_frame'],3) if isinstance(v,dict) else round(v,3)) for k,v in s.items() if isinstance(v,(dict,float))})"
done; done
