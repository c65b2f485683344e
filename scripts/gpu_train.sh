cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "train or generic or backward" > gpurun_out/pytest_train.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_train.log; grep -E "^E  |FAILED" gpurun_out/pytest_train.log | head
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_train.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_train.log').read().strip().splitlines()[-1]); t=d.get('training_step'); print({k:v for k,v in (t or {}).items() if k!='note'}); print('frame', d['ms_per_step'])"
