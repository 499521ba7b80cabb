# round-2 evidence on one GPU: full GPU tests, smoke, default bench, ncu launch list of the same command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g52_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g52_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g52_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g52_smoke.log
timeout 900 python bench.py > gpurun_out/g52_bench.log 2>&1; rc=$?; echo "bench rc=$rc"; tail -1 gpurun_out/g52_bench.log | cut -c1-160
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g52_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g52_ncu.log 2>&1; echo "ncu rc=$?"
