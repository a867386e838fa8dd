python tools/gpu/kab.py _variants/tr27/libusp.so --nz 1024 --iters 4 --rounds 1 2>&1 | grep -E "plane trace|variant" | tail -14
