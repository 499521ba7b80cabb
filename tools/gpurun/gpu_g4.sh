cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in split default; do
  for args in "1 2 60 0 0" "2 2 60 30 1" "1 4 12 0 0"; do
    SWF_ATTN=$k timeout 120 python tools/attn_diag.py $args >> gpurun_out/g4_diag.log 2>&1 || echo "rc=$? ($k $args)" >> gpurun_out/g4_diag.log
  done
done
cat gpurun_out/g4_diag.log
timeout 400 python -m pytest tests/test_gpu_group.py -k "backward or c4" -v -rA --timeout 200 > gpurun_out/g4_group.log 2>&1; echo "group rc=$?" >> gpurun_out/g4_diag.log
