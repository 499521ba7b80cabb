cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g73_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/g73_pytest.log
timeout 900 python bench.py > gpurun_out/g73_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g73_bench.log | cut -c1-120
