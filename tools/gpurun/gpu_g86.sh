# BF16 training mode, current code: ms per forward+backward call (tools/bwd_bench.py, 240x480, 2 blocks) and the
# ncu launch list of one call (serialised kernel time, to compare with the wall time per call).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -m gpu -q > gpurun_out/g86_t.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/g86_t.log)"
timeout 600 python tools/bwd_bench.py 240 480 3 > gpurun_out/g86_bwd.log 2>&1; echo "bwd_bench rc=$?"; cat gpurun_out/g86_bwd.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g86_launches.csv \
    python tools/bwd_once.py 240 480 > gpurun_out/g86_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/g86_launches.csv "BF16 training call 240x480" | head -40
