cd $GRAFT_REPO_ROOT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29841 tools/dp_diag2.py > gpurun_out/g16.log 2>&1
grep -E "wp2=|forward|Error" gpurun_out/g16.log
