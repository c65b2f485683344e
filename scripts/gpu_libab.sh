# A/B the bench over library variants: LIBS="v3x2 v6x1 ..." (paper_2103_13744_b200/_lib/var/libgf_*.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for v in ${LIBS}; do
  for rep in 1 2; do
  GF_DEBUG=1 GF_LIB_PATH=$PWD/paper_2103_13744_b200/_lib/var/libgf_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$v.log 2>&1 || tail -5 gpurun_out/bench_$v.log
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$v.log').read().strip().splitlines()[-1])
s=d['stage_roofline']; print('$v', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_frame'],3), {k:round(v['ms_per_frame'],3) for k,v in s.items() if isinstance(v, dict)}, 'Q', d['queries_per_frame'], 'clk', d['clocks']['sm_mhz'])"
  grep "k_mlp_tc" gpurun_out/bench_$v.log | sort -u | head -2
  done
done
