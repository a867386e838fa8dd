timeout 900 python -m pytest tests/test_gpu_xform.py tests/test_gpu_parity.py tests/test_gpu_slab.py -q 2>&1 | tail -2
P=paper_2207_14222_b200/libusp.so
timeout 600 python tools/gpu/kab.py $P $P:USP_LEAN=0 $P:USP_SPARSE_S=0 --config C5 --size 1024 --rounds 3 --iters 30 2>&1 | grep variant | cut -c1-250
