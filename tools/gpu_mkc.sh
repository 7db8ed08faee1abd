export EEB_SKIP_BUILD=1
timeout 120 python tools/mk_check.py 2>&1 | tail -20
timeout 120 python tools/mk_check.py gqa 2>&1 | tail -12
