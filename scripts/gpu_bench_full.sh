cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
( time timeout 900 python bench.py ) > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
cat gpurun_out/nproc.txt; tail -c 1500 gpurun_out/bench_full.log; tail -c 1200 gpurun_out/bench_ref.log
