cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -x -q > gpurun_out/g31_t.log 2>&1; echo "bwd_tc tests rc=$?"; tail -5 gpurun_out/g31_t.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or train or loss" > gpurun_out/g31_p.log 2>&1; echo "parity bwd rc=$?"; tail -2 gpurun_out/g31_p.log
timeout 900 python tools/bwd_bench.py 240 480 2 > gpurun_out/g31_bwd_mid.log 2>&1; echo "rc=$?"; cat gpurun_out/g31_bwd_mid.log
