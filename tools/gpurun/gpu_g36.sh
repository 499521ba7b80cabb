cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py tests/test_gpu_parity.py -q -k "bwd or backward or train or loss" > gpurun_out/g36_bwd.log 2>&1; echo "bwd tests rc=$?"; tail -3 gpurun_out/g36_bwd.log
timeout 900 python tools/bwd_bench.py 240 480 2 > gpurun_out/g36_bwd_mid.log 2>&1; echo "rc=$?"; cat gpurun_out/g36_bwd_mid.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g36_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/g36_pytest.log
