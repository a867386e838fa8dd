# z-quad K_C (8-column tiles, two CTAs per SM) vs the z-pair build:
# bit-identity tests with the variant library in place, then in-process A/B
mkdir -p gpurun_out
cp paper_2207_14222_b200/libusp.so /tmp/base_libusp.so
cp _variants/vq/libusp.so paper_2207_14222_b200/libusp.so
timeout 900 python -m pytest tests/test_gpu_zpair.py tests/test_gpu_real.py -q -x 2>&1 | tail -15 > gpurun_out/zq_tests.log
cp /tmp/base_libusp.so paper_2207_14222_b200/libusp.so
timeout 600 python tools/gpu/kab.py _variants/base/libusp.so _variants/vq/libusp.so --rounds 5 --iters 20 > gpurun_out/zq_ab_c5.log 2>&1
timeout 400 python tools/gpu/kab.py _variants/base/libusp.so _variants/vq/libusp.so --rounds 5 --iters 20 --config C4 --size 512 > gpurun_out/zq_ab_c4.log 2>&1
timeout 400 python tools/gpu/kab.py _variants/base/libusp.so _variants/vq/libusp.so --rounds 5 --iters 20 --opts delta_form=1 > gpurun_out/zq_ab_c5d.log 2>&1
echo done
