# final code on 2 GPUs: C4 (40B-shaped 2-block slice) with WP 1x2 and SP 2, and the C2 step with SP 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
i=0
for args in "--workload c4" "--workload c4 --sp 2" "--sp 2"; do
  i=$((i+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29670+i)) \
      bench.py --gpus 2 $args > gpurun_out/g91_$i.log 2>&1; echo "[$args] rc=$?"; grep '^{' gpurun_out/g91_$i.log | tail -1 | cut -c1-220
done
