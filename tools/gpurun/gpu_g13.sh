cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/dp_diag.py > gpurun_out/g13.log 2>&1
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29811 tools/dp_diag.py >> gpurun_out/g13.log 2>&1
SWF_DIAG_SERIAL=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29812 tools/dp_diag.py >> gpurun_out/g13.log 2>&1
OMP_NUM_THREADS=1 timeout 200 python tools/dp_diag.py >> gpurun_out/g13.log 2>&1
grep "^rank" gpurun_out/g13.log
timeout 900 python -m pytest tests/test_gpu_group.py -v --timeout 300 -k "wp2x4 or c4 or train or backward" > gpurun_out/g13_group.log 2>&1; echo "group rc=$?"; grep -E "PASSED|FAILED" gpurun_out/g13_group.log
