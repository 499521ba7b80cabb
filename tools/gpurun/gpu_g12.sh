# full GPU test suite (per-file logs, per-test timeouts) + default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "1 2 60 0 0" "2 2 60 30 1"; do
  timeout 120 python tools/attn_diag.py $args >> gpurun_out/g12_diag.log 2>&1
done
cat gpurun_out/g12_diag.log
timeout 2400 python -m pytest tests -m gpu -v -rfE --timeout 600 --durations=30 > gpurun_out/g12_pytest.log 2>&1
echo "pytest rc=$?"; tail -40 gpurun_out/g12_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g12_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/g12_smoke.log | tail -2
timeout 900 python bench.py > gpurun_out/g12_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/g12_bench.log | tail -1 | head -c 1500
