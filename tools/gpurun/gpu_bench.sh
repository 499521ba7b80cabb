# Bench line (1 GPU, C2) plus the ncu launch list of the same command.
# usage: bash tools/gpurun/gpu_bench.sh TAG
T=${1:-bench}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/${T}_bench.log | tail -1
