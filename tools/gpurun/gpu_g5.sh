cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in MID H1K C4W1 C4W; do
  for k in split default; do
    SWF_ATTN=$k timeout 150 python tools/sp_diag.py $c >> gpurun_out/g5_sp.log 2>&1 || echo "rc=$? ($c $k)" >> gpurun_out/g5_sp.log
  done
done
cat gpurun_out/g5_sp.log
