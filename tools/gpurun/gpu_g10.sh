# A/B of attention build variants (kernel isolation, live weights) + QKV epilogue staging
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in pb40 pb256 pb1000 pb256p3 pb256p1; do
  echo "== $v" >> gpurun_out/g10_ab.log
  SWF_LIB=paper_2509_13523_b200/_build_variants/$v.so timeout 200 python tools/kbench.py 10 attention >> gpurun_out/g10_ab.log 2>&1
done
for v in oldqkv pb256; do
  echo "== qkv $v" >> gpurun_out/g10_ab.log
  SWF_LIB=paper_2509_13523_b200/_build_variants/$v.so timeout 200 python tools/kbench.py 10 qkv_gemm >> gpurun_out/g10_ab.log 2>&1
done
done
cat gpurun_out/g10_ab.log
