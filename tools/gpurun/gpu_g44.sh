cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g44_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g44_bench.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g44_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g44_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/g44_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/g44_ref.log | cut -c1-300
