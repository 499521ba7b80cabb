cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SWF_PREC=fp32 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29831 tools/wp_check.py > gpurun_out/g15.log 2>&1
SWF_PREC=fp32 SWF_OWN=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29832 tools/wp_check.py >> gpurun_out/g15.log 2>&1
grep -E "C1:|MID|WP_CHECK|Error|rank" gpurun_out/g15.log | head -30
