set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r12_tests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/r12_tests.log
timeout 900 python bench.py > gpurun_out/r12_bench.log 2>&1; echo "bench rc=$?"
tail -c 800 gpurun_out/r12_bench.log
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches.csv python bench.py > gpurun_out/r12_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r12_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn|k_gemm_tc" -s 8 -c 6 -o gpurun_out/r12_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r12_ncu_full.log 2>&1; echo "ncu full rc=$?"
