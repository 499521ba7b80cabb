# BF16 training mode: 8 worker streams for the per-plane attention-backward GEMMs (was 4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py -m gpu -q -x > gpurun_out/g94_t.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/g94_t.log)"
timeout 600 python tools/bwd_bench.py 240 480 3 > gpurun_out/g94_bwd.log 2>&1; echo "bwd_bench rc=$?"; cat gpurun_out/g94_bwd.log
timeout 900 python bench.py --workload train --train-precision bf16 > gpurun_out/g94_train_bf16.log 2>&1; echo "train rc=$?"; tail -1 gpurun_out/g94_train_bf16.log | cut -c1-200
