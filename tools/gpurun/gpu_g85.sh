# out-projection + encode epilogues in 16-byte pieces through shared memory (epi32_v4):
# full GPU tests + smoke on the working tree, then default bench runs alternating with HEAD's library.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g85_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/g85_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g85_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g85_smoke.log
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernels',{})
print(sys.argv[2], round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {n: round(v['ms_per_launch'],2) if isinstance(v,dict) else v for n,v in k.items()})" $1 $2; }
for r in 1 2; do
  timeout 900 python bench.py > gpurun_out/g85_new$r.log 2>&1; echo "new rc=$?"; summ gpurun_out/g85_new$r.log new$r
  SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/q_base.so timeout 900 python bench.py > gpurun_out/g85_base$r.log 2>&1; echo "base rc=$?"; summ gpurun_out/g85_base$r.log base$r
done
