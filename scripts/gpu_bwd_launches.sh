cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for v in GF_BWD_TC=1 GF_BWD_TC=0; do
env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_grouped_backward|k_bwd" \
  --log-file gpurun_out/bwd_launches_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --clock-preroll 0 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/bwd_launches_$v.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki][:40], r[mi])].append(float(r[vi].replace(',','')))
for k,v in sorted(agg.items()): print('$v', k, len(v), sum(v)/len(v))
PY
done
