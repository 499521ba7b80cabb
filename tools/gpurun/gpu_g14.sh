cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SWF_DP_WP=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29821 tools/dp_check.py > gpurun_out/g14.log 2>&1
SWF_TRAIN_VERBOSE=1 SWF_DP_WP=2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29822 tools/dp_check.py >> gpurun_out/g14.log 2>&1
grep -E "mb_losses|world=|PASS|FAIL|Error" gpurun_out/g14.log
