export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for dbg in 0 64 128; do
EEB_MK=1 EEB_MK_DBG=$dbg EEB_MK_TRACE=gpurun_out/st.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo "dbg=$dbg"; python tools/mk_trace_step.py gpurun_out/st.bin 2>/dev/null | grep -E "norm|gemm|step"
done
