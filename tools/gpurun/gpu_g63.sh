cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_parity.py tests/test_gpu_group.py -x -q > gpurun_out/g63_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g63_t.log
bash tools/gpurun/gpu_hbm.sh
