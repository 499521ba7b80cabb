timeout 300 python tools/kbench.py 10 gateup_gemm,down_gemm,qkv_gemm,out_gemm > gpurun_out/r21_kbench.log 2>&1; cat gpurun_out/r21_kbench.log | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r21_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r21_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r21_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/r21_bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['tflops_per_gpu'], d['clocks'])
for k,v in d['kernels'].items(): print(k, round(v['ms_per_launch'],2), v['tflops'])
"
