# final-code evidence on one GPU: full GPU tests, smoke, two default bench runs, the ncu launch list of
# the bench command, and ncu --set full of one launch of each GEMM + the attention (traffic bytes)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g89_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g89_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g89_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g89_smoke.log
for r in 1 2; do timeout 900 python bench.py > gpurun_out/g89_bench$r.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g89_bench$r.log | cut -c1-120; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g89_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g89_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none -k regex:"k_gemm_tc|k_attn_pp" -s 22 -c 5 \
    -o gpurun_out/g89_full -f python tools/kbench.py 2 qkv_gemm > gpurun_out/g89_full.log 2>&1; echo "ncu full rc=$?"
