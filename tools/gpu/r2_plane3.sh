timeout 900 python -m pytest tests/test_gpu_plane.py -x -q 2>&1 | tail -5
cp paper_2207_14222_b200/libusp.so _variants/y31.so
python tools/gpu/kab.py _variants/y22/libusp.so _variants/y27/libusp.so _variants/y31.so _variants/y36/libusp.so _variants/y41/libusp.so --nz 256 --iters 20 --rounds 3
