cd $GRAFT_REPO_ROOT
cd _r1 && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29851 dp_diag2.py > ../gpurun_out/g17.log 2>&1
cd ..; grep -E "wp2=|forward|Error" gpurun_out/g17.log
