cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g49_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g49_bench.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/g49_bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g49_bench2.log | cut -c1-200
