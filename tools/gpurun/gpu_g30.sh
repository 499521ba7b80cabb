cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/bwd_bench.py 120 240 3 > gpurun_out/g30_bwd_small.log 2>&1; echo "rc=$?"; cat gpurun_out/g30_bwd_small.log
timeout 900 python tools/bwd_bench.py 240 480 2 > gpurun_out/g30_bwd_mid.log 2>&1; echo "rc=$?"; cat gpurun_out/g30_bwd_mid.log
