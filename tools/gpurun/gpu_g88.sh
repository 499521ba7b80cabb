# BF16 training mode: column sums over token slices, gate/up recompute product written directly (no epilogue pass)
# row statistics: training-mode tests, then ms per call and the launch list (compare tools/gpurun/gpu_g86.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_tc.py tests/test_gpu_parity.py tests/test_gpu_group.py -m gpu -q -x > gpurun_out/g88_t.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/g88_t.log)"
timeout 600 python tools/bwd_bench.py 240 480 3 > gpurun_out/g88_bwd.log 2>&1; echo "bwd_bench rc=$?"; cat gpurun_out/g88_bwd.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g88_launches.csv \
    python tools/bwd_once.py 240 480 > gpurun_out/g88_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/g88_launches.csv "BF16 training call 240x480" 2>/dev/null | head -20
for p in bf16 fp32; do timeout 900 python bench.py --workload train --train-precision $p > gpurun_out/g88_train_$p.log 2>&1; echo "train $p rc=$?"; tail -1 gpurun_out/g88_train_$p.log | cut -c1-300; done
