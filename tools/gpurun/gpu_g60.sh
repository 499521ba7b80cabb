cd $GRAFT_REPO_ROOT; timeout 120 ./tools/_mma2_probe
