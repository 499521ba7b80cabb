cd $GRAFT_REPO_ROOT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29871 tools/dp_diag2.py > gpurun_out/g19.log 2>&1
grep -E "wp2=|forward|Error" gpurun_out/g19.log
timeout 900 python -m pytest tests/test_gpu_wp.py tests/test_gpu_group.py -v --timeout 300 > gpurun_out/g19_wp.log 2>&1; echo "rc=$?"; grep -E "PASSED|FAILED" gpurun_out/g19_wp.log | grep -v "forward_bitwise" ; tail -3 gpurun_out/g19_wp.log
