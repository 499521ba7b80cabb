set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r7_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r7_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r7_bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/r7_bench.log
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r7_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 4 -c 1 -o gpurun_out/r7_attn python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r7_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
