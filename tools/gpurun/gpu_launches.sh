# GPU test suite + smoke + default bench + ncu launch list of the same bench command.
# usage: bash tools/gpurun/gpu_launches.sh TAG
T=${1:-launch}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_plain.log 2>&1; rc=$?; echo "plain bench rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
