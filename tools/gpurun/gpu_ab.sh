# A/B of an environment switch on kernel-isolation timings. usage: bash tools/gpurun/gpu_ab.sh TAG VAR classes
T=$1; V=$2; K=${3:-gateup_gemm,down_gemm,qkv_gemm,out_gemm}
timeout 300 python tools/kbench.py 30 $K > gpurun_out/${T}_a.log 2>&1; echo "A rc=$?"; cat gpurun_out/${T}_a.log
env $V=1 timeout 300 python tools/kbench.py 30 $K > gpurun_out/${T}_b.log 2>&1; echo "B ($V) rc=$?"; cat gpurun_out/${T}_b.log
