timeout 600 python tools/kbench.py 10 > gpurun_out/r11_kbench.log 2>&1; echo "kbench rc=$?"
cat gpurun_out/r11_kbench.log | tail -12
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r11_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r11_tests.log
