cd $GRAFT_REPO_ROOT
bash tools/gpurun/gpu_hbm.sh
timeout 900 python tools/grid_scaling.py > gpurun_out/grid_scaling.log 2>&1; echo "grid rc=$?"; cat gpurun_out/grid_scaling.log | tail -4
