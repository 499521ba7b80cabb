set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r3_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r3_tests.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r3_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r3_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 2 -c 1 -o gpurun_out/r3_attn python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 30 -c 2 -o gpurun_out/r3_gemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
ls -la gpurun_out
