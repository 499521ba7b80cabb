# Round-end validation on a 2-GPU box: GPU tests, smoke, the default bench, and the C5 / training
# workloads on 2 GPUs. usage: bash tools/gpurun/gpu_final.sh TAG
T=${1:-final}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${T}_bench.log | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
    bench.py --gpus 2 --workload c5 --members 4 > gpurun_out/${T}_c5.log 2>&1; echo "c5 rc=$?"; grep '^{' gpurun_out/${T}_c5.log | tail -1 | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 \
    bench.py --gpus 2 --workload train --steps 2 --warmup 3 > gpurun_out/${T}_train2.log 2>&1; echo "train2 rc=$?"; grep '^{' gpurun_out/${T}_train2.log | tail -1 | cut -c1-200
