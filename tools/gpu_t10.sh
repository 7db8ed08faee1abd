export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for xs in 4 12 16 20; do
EEB_MK=1 EEB_MK_XSTAGES=$xs EEB_MK_TRACE=gpurun_out/st.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo "xs=$xs"; python tools/mk_trace_step.py gpurun_out/st.bin 2>/dev/null | grep -E "gemm|step"
done
