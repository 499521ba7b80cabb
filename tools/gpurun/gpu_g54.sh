cd $GRAFT_REPO_ROOT; timeout 120 ./tools/_mma2_probe; timeout 120 ./tools/_mma_probe | grep -E "N64|SS N128  "
