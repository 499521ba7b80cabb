cd $GRAFT_REPO_ROOT
for s in 1 2; do echo "== sites $s"; SWF_DBG_TC=$s timeout 300 python tools/bwd_err_probe.py 2>&1 | tail -3; done
for mo in 1 2 4 8 16 32; do echo "== fwd modes $mo"; SWF_DBG_TC=1 SWF_DBG_MODES=$mo timeout 300 python tools/bwd_err_probe.py 2>&1 | tail -1; done
