cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in a_hint a_b0; do
  SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/$v.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/g24_t_$v.log 2>&1; echo "tests $v rc=$?"; tail -1 gpurun_out/g24_t_$v.log
done
bash tools/gpurun/gpu_var_cycles.sh g24 attention k_attn_pp
