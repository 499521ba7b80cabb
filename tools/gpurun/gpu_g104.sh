# dS epilogue: P rows loaded through the shared-memory staging (8 lines per load): training tests, benches, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_tc.py tests/test_gpu_parity.py tests/test_gpu_group.py -m gpu -q -x > gpurun_out/g104_t.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/g104_t.log)"
timeout 600 python tools/bwd_bench.py 240 480 3 > gpurun_out/g104_bwd.log 2>&1; echo "bwd_bench rc=$?"; cat gpurun_out/g104_bwd.log
timeout 900 python bench.py --workload train --train-precision bf16 > gpurun_out/g104_train_bf16.log 2>&1; echo "train rc=$?"; tail -1 gpurun_out/g104_train_bf16.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g104_launches.csv \
    python tools/bwd_once.py 240 480 > gpurun_out/g104_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/g104_launches.csv "BF16 training call 240x480" 2>/dev/null | head -16
