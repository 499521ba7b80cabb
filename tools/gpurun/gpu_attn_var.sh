# Attention build variants (paper_2509_13523_b200/_build/var/lib_*.so via SWF_LIB): kernel isolation
# time and energy, repeated twice in alternating order. usage: bash tools/gpurun/gpu_attn_var.sh TAG
T=${1:-av}
for rep in 1 2; do
  for lib in paper_2509_13523_b200/_build/var/lib_*.so; do
    v=$(basename $lib .so)
    SWF_LIB=$PWD/$lib timeout 300 python tools/kbench.py 20 attention > gpurun_out/${T}_${v}_$rep.log 2>&1
    echo "$v rep$rep rc=$? $(grep -o '"ms": [0-9.]*\|J_per_launch": [0-9.]*\|"sm_mhz": [0-9.]*' gpurun_out/${T}_${v}_$rep.log | tr '\n' ' ')"
  done
done
