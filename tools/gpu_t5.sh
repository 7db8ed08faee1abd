export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for cfg in "0 0" "4 0" "0 3"; do set -- $cfg
EEB_MK=1 EEB_MK_DBG=$1 EEB_MK_WSTAGES=$2 EEB_MK_TRACE=gpurun_out/st.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo "dbg=$1 wstages=$2"; python tools/mk_trace_step.py gpurun_out/st.bin 2>/dev/null
done
