cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "MID load sp2" "MID init sp2" "MID init wp2" "MID load wp2"; do
  timeout 100 python tools/sp_diag.py $a >> gpurun_out/g7_sp.log 2>&1 || echo "rc=$? ($a)" >> gpurun_out/g7_sp.log
done
cat gpurun_out/g7_sp.log
bash tools/gpurun/gpu_g6.sh
