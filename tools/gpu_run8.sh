set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r8_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r8_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r8_bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/r8_bench.log
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r8_plain.log 2>&1 && \
