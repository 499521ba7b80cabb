for i in 1 2; do
timeout 300 python tools/kbench.py 10 attention > gpurun_out/r15_v3_$i.log 2>&1; tail -1 gpurun_out/r15_v3_$i.log
SWF_LIB=paper_2509_13523_b200/_build_v2/libswinflow_b200.so timeout 300 python tools/kbench.py 10 attention > gpurun_out/r15_v2_$i.log 2>&1; tail -1 gpurun_out/r15_v2_$i.log
done
