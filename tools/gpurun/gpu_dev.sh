# Development loop on one B200: attention smoke, GPU parity tests, kernel-isolation timings.
# usage: bash tools/gpurun/gpu_dev.sh TAG
T=${1:-dev}
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_bf16" > gpurun_out/${T}_c1.log 2>&1; rc=$?; echo "c1 rc=$rc"; tail -2 gpurun_out/${T}_c1.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
timeout 300 python tools/kbench.py 10 > gpurun_out/${T}_kbench.log 2>&1; echo "kbench rc=$?"; cat gpurun_out/${T}_kbench.log
