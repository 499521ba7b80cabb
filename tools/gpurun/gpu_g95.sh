# BF16 training step: ncu launch list (device time per step, serialised) vs the bench's wall time per step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g95_launches.csv \
    python bench.py --workload train --train-precision bf16 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g95_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/g95_launches.csv "BF16 training step" 2>/dev/null | head -24
