# ncu evidence for profiles/: launch list of the default bench command, and a full capture of the
# attention kernel and of the GEMMs (one step). usage: bash tools/gpurun/gpu_profile.sh TAG
T=${1:-prof}
timeout 900 python bench.py > gpurun_out/${T}_plain.log 2>&1; rc=$?; echo "plain bench rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_short.log 2>&1; echo "short rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_attn_tc|k_gemm_tc" -s 9 -c 6 \
    -o gpurun_out/${T}_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
