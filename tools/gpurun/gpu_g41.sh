cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload train --train-precision bf16 --steps 2 --warmup 1 > gpurun_out/g41_train_bf16.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/g41_train_bf16.log | cut -c1-400
timeout 900 python bench.py --workload train --steps 1 --warmup 1 > gpurun_out/g41_train_fp32.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/g41_train_fp32.log | cut -c1-400
