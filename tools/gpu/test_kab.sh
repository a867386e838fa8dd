# GPU suite + in-process A/B of the given variants against the product build
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/gpu/kab.py "$@" 2>&1 | grep -v Warning
