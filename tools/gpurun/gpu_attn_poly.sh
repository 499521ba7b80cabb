# A/B of the share of exponentials on the FMA pipe (SWF_ATTN_POLY8 of 8)
for pv in ${POLYS:-0 1 2 0 1 2}; do
  cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make EXTRA="-DSWF_ATTN_POLY8=$pv" > /dev/null 2>&1; cd ..
  timeout 200 python tools/kbench.py 20 attention > gpurun_out/poly$pv.log 2>&1; echo "poly $pv/8: $(tail -1 gpurun_out/poly$pv.log | cut -c1-160)"
done
cd paper_2509_13523_b200 && touch csrc/k_attn.cu && make > /dev/null 2>&1; cd ..
