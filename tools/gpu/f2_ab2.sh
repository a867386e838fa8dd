# paired fp32, second round: v3 = paired everywhere + paired K_C multiplier (no spill),
# v4 = v3 with scalar DFT butterflies (paired complex multiply / axpy only)
mkdir -p gpurun_out
timeout 600 python tools/gpu/kab.py _variants/base/libusp.so _variants/v3/libusp.so _variants/v4/libusp.so --rounds 5 --iters 20 > gpurun_out/f2b_ab_c5.log 2>&1
timeout 400 python tools/gpu/kab.py _variants/base/libusp.so _variants/v3/libusp.so _variants/v4/libusp.so --rounds 5 --iters 20 --config C4 --size 512 > gpurun_out/f2b_ab_c4.log 2>&1
echo done
