export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for cfg in "0 4" "16 4" "32 4" "16 12" "32 12"; do set -- $cfg
EEB_MK=1 EEB_MK_L2=$1 EEB_MK_XSTAGES=$2 EEB_MK_TRACE=gpurun_out/st.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo "l2=$1 xs=$2"; python tools/mk_trace_step.py gpurun_out/st.bin 2>/dev/null | grep -E "gemm|step"
done
