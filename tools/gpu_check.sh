set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or fp32 or nan or noise" > gpurun_out/r1_fp32.log 2>&1; echo "fp32 rc=$?"
tail -30 gpurun_out/r1_fp32.log
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "selftest" > gpurun_out/r1_gemm.log 2>&1; echo "gemm rc=$?"
tail -30 gpurun_out/r1_gemm.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "bf16 or locality" > gpurun_out/r1_bf16.log 2>&1; echo "bf16 rc=$?"
tail -40 gpurun_out/r1_bf16.log
