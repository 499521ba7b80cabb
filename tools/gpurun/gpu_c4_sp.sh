# C4 (40B-shaped 2-block slice) with WP and SP on 2 GPUs, and the C2 step with SP 2.
T=${1:-c4}
for args in "--workload c4" "--workload c4 --sp 2" "--sp 2"; do
  tag=$(echo $args | tr -d ' -')
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 \
      bench.py --gpus 2 $args > gpurun_out/${T}_$tag.log 2>&1; echo "$args rc=$?"; grep '^{' gpurun_out/${T}_$tag.log | tail -1 | cut -c1-160
done
