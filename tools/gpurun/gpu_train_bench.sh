# f3 measurement: FP32 training-step bench on a small grid slice, then its ncu launch list.
T=${1:-trainb}; G=${2:-"60 120"}
timeout 900 python bench.py --workload train --train-grid $G --steps 1 --warmup 3 > gpurun_out/${T}_plain.log 2>&1; rc=$?
echo "plain rc=$rc"; tail -2 gpurun_out/${T}_plain.log
[ $rc -eq 0 ] || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --workload train --train-grid $G --steps 1 --warmup 3 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
