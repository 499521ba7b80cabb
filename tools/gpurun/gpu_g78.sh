cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g78_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/g78_pytest.log
timeout 900 python bench.py > gpurun_out/g78_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g78_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['roofline']['frac'], {a:round(b['ms_per_launch'],2) for a,b in k.items()}, round(d['e2e']['value']))"
