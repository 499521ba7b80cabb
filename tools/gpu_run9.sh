timeout 600 python tools/kbench.py 10 > gpurun_out/r9_kbench.log 2>&1; echo "kbench rc=$?"
cat gpurun_out/r9_kbench.log | tail -12
