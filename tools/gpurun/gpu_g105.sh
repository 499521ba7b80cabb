# attention lazy-rescale threshold 2^8 (a_r08, current) vs 2^12 (a_r12): attention tests on a_r12, base-clock
# cycles and free-clock ms of the attention kernel (live weights)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/a_r12.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_c2_spot.py -m gpu -q > gpurun_out/g105_t.log 2>&1; echo "tests(a_r12) rc=$? $(tail -1 gpurun_out/g105_t.log)"
bash tools/gpurun/gpu_var_cycles.sh g105 attention 'k_attn_pp' > /dev/null 2>&1
cat gpurun_out/g105_cyc.log
