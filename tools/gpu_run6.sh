set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r6_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r6_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r6_bench.log 2>&1; echo "bench rc=$?"
tail -c 1800 gpurun_out/r6_bench.log
