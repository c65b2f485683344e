# training backward: tests, bench side measurement, launch list and ncu --set full of the backward kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_train.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_train.log; grep -E "^E  |FAILED" gpurun_out/pytest_train.log | head
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_train.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_train.log').read().strip().splitlines()[-1]); t=d.get('training_step'); print({k:v for k,v in (t or {}).items() if k!='note'}); print('frame', d['ms_per_step'])" || tail -5 gpurun_out/bench_train.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_grouped_backward|k_bwd|k_group_|k_adam|k_photo|k_prep" \
  --log-file gpurun_out/bwd_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/bwd_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki][:40], r[mi])].append(float(r[vi].replace(',','')))
for k,v in sorted(agg.items()): print(k, len(v), sum(v)/len(v))
PY
for k in ${PROF_KERNELS}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
  -o gpurun_out/prof_bwd_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1; echo "ncu $k rc=$?"
done
