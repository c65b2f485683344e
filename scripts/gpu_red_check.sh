cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
bash scripts/gpu_prof_reduce.sh
