# A/B of diagnostic library variants (timing only; results are garbage).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in base ${EXPS:-1 3}; do
  if [ $v = base ]; then lib=""; else lib=$PWD/paper_2103_13744_b200/_lib/exp/lib$v.so; fi
  GF_LIB_PATH=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/exp_$v.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/exp_$v.log') if l.startswith('{')][-1]); print('$v', round(d['ms_per_step'],3), {k:(round(v['ms_per_frame'],3)) for k,v in d['stage_roofline'].items()})" || tail -3 gpurun_out/exp_$v.log
done
