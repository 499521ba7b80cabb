cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_sampler.py tests/test_gpu_c2_spot.py -q -rA 2>&1 | tail -60 > gpurun_out/g1_tests.log
cat gpurun_out/g1_tests.log | tail -60
