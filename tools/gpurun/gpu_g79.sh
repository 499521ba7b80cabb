cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_tc.py tests/test_gpu_group.py tests/test_gpu_wp.py -q > gpurun_out/g79_t.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/g79_t.log
