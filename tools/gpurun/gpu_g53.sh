cd $GRAFT_REPO_ROOT; timeout 300 ./tools/_mma_probe
