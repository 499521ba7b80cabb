cd $GRAFT_REPO_ROOT
for dbg in 0 1 4 5; do
  echo "== SWF_DBG=$dbg" >> gpurun_out/g18.log
  SWF_DBG=$dbg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2986$dbg tools/dp_diag2.py > gpurun_out/g18_$dbg.log 2>&1
  grep -E "wp2=|forward|Error" gpurun_out/g18_$dbg.log >> gpurun_out/g18.log
done
cat gpurun_out/g18.log
