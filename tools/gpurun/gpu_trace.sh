# Attention pipeline trace (development build with clock64 stamps; see k_attn.cu SWF_ATTN_TRACE).
# usage: bash tools/gpurun/gpu_trace.sh ["-DSWF_ATTN_NOSOFTMAX"]
cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make EXTRA="-DSWF_ATTN_TRACE $1" > /dev/null 2>&1; cd ..
SWF_ATTN_TRACE_OUT=gpurun_out/attn_trace.bin timeout 200 python tools/kbench.py 2 attention > gpurun_out/trace_kbench.log 2>&1
echo "trace rc=$?"; tail -1 gpurun_out/trace_kbench.log
python tools/attn_trace.py gpurun_out/attn_trace.bin 29 0
cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make > /dev/null 2>&1; cd ..
