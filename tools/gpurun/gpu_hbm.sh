# ncu evidence for the HBM-bound kernels: DRAM bytes and duration per launch (C2 forecast step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/hbm_probe.py > gpurun_out/hbm_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_gather|k_scatter|k_sampler|k_fold|k_noise|k_inv_rms|k_build|k_assemble|k_standard|k_destd|k_churn|k_time|k_ada|k_peer" \
  -c 3000 --csv python tools/hbm_probe.py > gpurun_out/hbm_ncu.csv 2> gpurun_out/hbm_ncu.err; echo "ncu rc=$?"
python tools/ncu_hbm_summary.py gpurun_out/hbm_ncu.csv | tee gpurun_out/hbm_summary.txt
