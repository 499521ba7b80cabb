cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_c2_spot.py tests/test_gpu_bwd_tc.py -x -q > gpurun_out/g68_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g68_t.log
timeout 900 python bench.py > gpurun_out/g68_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g68_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {a:round(b['ms_per_launch'],2) for a,b in k.items()}, round(d['e2e']['value']))"
