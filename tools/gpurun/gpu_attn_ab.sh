# A/B of the attention softmax split (SWF_ATTN_SPLIT 2 vs 4): kernel-isolation time, energy, trace.
for sp in 2 4 2 4; do
  cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make EXTRA="-DSWF_ATTN_SPLIT=$sp" > /dev/null 2>&1; cd ..
  timeout 200 python tools/kbench.py 20 attention > gpurun_out/ab_split$sp.log 2>&1; echo "split $sp: $(tail -1 gpurun_out/ab_split$sp.log)"
done
cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make EXTRA="-DSWF_ATTN_TRACE -DSWF_ATTN_SPLIT=4" > /dev/null 2>&1; cd ..
SWF_ATTN_TRACE_OUT=gpurun_out/attn_trace4.bin timeout 200 python tools/kbench.py 2 attention > /dev/null 2>&1
python tools/attn_trace.py gpurun_out/attn_trace4.bin 29 0 | grep -v "^item"
cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make > /dev/null 2>&1; cd ..
