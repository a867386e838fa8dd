# in-process A/B of library variants (tools/gpu/kab.py); args passed through
timeout 900 python tools/gpu/kab.py "$@" 2>&1 | grep -v Warning
