cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/bwd_err_probe.py 0.03 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -q > gpurun_out/g39_t.log 2>&1; echo "bwd_tc tests rc=$?"; tail -3 gpurun_out/g39_t.log
timeout 900 python tools/bwd_bench.py 240 480 2 > gpurun_out/g39_bwd_mid.log 2>&1; echo "rc=$?"; cat gpurun_out/g39_bwd_mid.log
