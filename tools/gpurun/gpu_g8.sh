cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "1 2 60 0 0" "2 2 60 30 1" "1 4 12 0 0" "2 4 8 4 1"; do
  timeout 120 python tools/attn_diag.py $args >> gpurun_out/g8_diag.log 2>&1 || echo "rc=$? ($args)" >> gpurun_out/g8_diag.log
done
cat gpurun_out/g8_diag.log
for a in "MID load sp2" "MID init sp2" "C4W init sp2" "MID load wp2"; do
  timeout 100 python tools/sp_diag.py $a >> gpurun_out/g8_sp.log 2>&1 || echo "rc=$? ($a)" >> gpurun_out/g8_sp.log
done
cat gpurun_out/g8_sp.log
for k in default split; do
  echo "== $k" >> gpurun_out/g8_ab.log
  SWF_ATTN=$k timeout 300 python tools/kbench.py 10 attention >> gpurun_out/g8_ab.log 2>&1
done
cat gpurun_out/g8_ab.log
