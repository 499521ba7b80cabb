cd $GRAFT_REPO_ROOT
timeout 300 python tools/bwd_err_probe.py 0.03 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -q > gpurun_out/g34_t.log 2>&1; echo "bwd_tc tests rc=$?"; tail -5 gpurun_out/g34_t.log
