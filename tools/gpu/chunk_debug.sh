for g in 0 8; do echo "G=$g"; USP_CHUNK=$g python tools/gpu/chunk_debug.py 128,128,128 > gpurun_out/cd$g.txt 2>&1; tail -3 gpurun_out/cd$g.txt; done
USP_CHUNK=8 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "closed_form and shape12" 2>&1 | grep -E "Error|assert|err" | head -20
