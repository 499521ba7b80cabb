# round-2 parity checks, one file at a time with per-test timeouts (logs stream into gpurun_out/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/g2_nproc.log
run() {  # name, wall limit, per-test limit, pytest args...
  n=$1; lim=$2; per=$3; shift 3
  timeout $lim python -m pytest "$@" -v -rA --timeout $per --durations=0 > gpurun_out/g2_$n.log 2>&1
  echo "$n rc=$?" >> gpurun_out/g2_summary.log
}
run attn 240 120 tests/test_gpu_attention.py
run samp 300 150 tests/test_gpu_sampler.py
run bw 200 100 tests/test_gpu_parity.py -k block_window
run group 600 200 tests/test_gpu_group.py
run cpp 200 150 tests/test_cpp_api.py
run c2 600 400 tests/test_gpu_c2_spot.py
run depth 300 200 tests/test_gpu_depth.py
cat gpurun_out/g2_summary.log
