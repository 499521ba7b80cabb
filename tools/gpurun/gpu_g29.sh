cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -x -q > gpurun_out/g29_t.log 2>&1; echo "bwd_tc tests rc=$?"; tail -30 gpurun_out/g29_t.log
