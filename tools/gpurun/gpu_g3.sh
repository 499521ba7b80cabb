# attention self-test (rescale fix), group backward + C4-width SP, C2 per-block increments
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, wall limit, per-test limit, pytest args...
  n=$1; lim=$2; per=$3; shift 3
  timeout $lim python -m pytest "$@" -v -rA --timeout $per --durations=0 > gpurun_out/g3_$n.log 2>&1
  echo "$n rc=$?" >> gpurun_out/g3_summary.log
}
run attn_small 120 60 tests/test_gpu_attention.py -k "small or fp32"
run attn 300 120 tests/test_gpu_attention.py
run samp 200 100 tests/test_gpu_sampler.py
run group 500 250 tests/test_gpu_group.py -k "backward or c4"
run c2 600 400 tests/test_gpu_c2_spot.py
cat gpurun_out/g3_summary.log
