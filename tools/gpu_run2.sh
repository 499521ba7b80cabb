set -x
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "t_range or solve_pf" > gpurun_out/r2_dbg.log 2>&1; echo "dbg rc=$?"
tail -30 gpurun_out/r2_dbg.log
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench.log
