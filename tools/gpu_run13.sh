timeout 600 python tools/kbench.py 10 attention,attention > gpurun_out/r13_kbench.log 2>&1; echo "kbench rc=$?"; cat gpurun_out/r13_kbench.log | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r13_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r13_tests.log
