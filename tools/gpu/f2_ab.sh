# paired-fp32 (FFMA2 / FADD2 / FMUL2) complex arithmetic vs the scalar build:
# parity tests with the new library in place, then in-process A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zpair.py tests/test_gpu_real.py -q -x 2>&1 | tail -15 > gpurun_out/f2_tests.log
timeout 600 python tools/gpu/kab.py _variants/base/libusp.so _variants/v2/libusp.so --rounds 5 --iters 20 > gpurun_out/f2_ab_c5.log 2>&1
timeout 400 python tools/gpu/kab.py _variants/base/libusp.so _variants/v2/libusp.so --rounds 5 --iters 20 --opts delta_form=1 > gpurun_out/f2_ab_c5d.log 2>&1
timeout 400 python tools/gpu/kab.py _variants/base/libusp.so _variants/v2/libusp.so --rounds 5 --iters 20 --config C4 --size 512 > gpurun_out/f2_ab_c4.log 2>&1
echo done
