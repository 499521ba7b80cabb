nvidia-smi topo -m | head -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/wp_check.py > gpurun_out/r10_wp.log 2>&1; echo "wp rc=$?"
tail -8 gpurun_out/r10_wp.log
SWF_OWN=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/wp_check.py > gpurun_out/r10_wp_rr.log 2>&1; echo "wp rr rc=$?"
tail -4 gpurun_out/r10_wp_rr.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/r10_bench2.log 2>&1; echo "bench2 rc=$?"
tail -c 1200 gpurun_out/r10_bench2.log
