# BF16 training mode at C2 widths vs the FP32 validation mode (new test), plus the rest of the training tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_tc.py -m gpu -q -x > gpurun_out/g92_t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g92_t.log
