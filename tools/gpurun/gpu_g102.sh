# last validation of the committed code: full GPU tests, smoke, one default bench run
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g102_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/g102_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g102_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g102_smoke.log
timeout 900 python bench.py > gpurun_out/g102_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g102_bench.log | cut -c1-160
timeout 900 python bench.py --workload train --train-precision bf16 > gpurun_out/g102_train.log 2>&1; echo "train rc=$?"; tail -1 gpurun_out/g102_train.log | cut -c1-160
