cd $GRAFT_REPO_ROOT; timeout 600 python tools/bwd_err_probe.py
