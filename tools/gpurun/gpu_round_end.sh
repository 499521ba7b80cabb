# Round-end evidence on a 2-GPU box: GPU tests, smoke, the default bench line, and the ncu launch
# list of the same bench command (after it exited 0). usage: bash tools/gpurun/gpu_round_end.sh TAG
T=${1:-end}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; rc=$?; echo "bench rc=$rc"; tail -1 gpurun_out/${T}_bench.log | cut -c1-200
[ $rc -eq 0 ] || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
