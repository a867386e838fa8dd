P=paper_2207_14222_b200/libusp.so
timeout 600 python tools/gpu/kab.py $P $P:USP_TSTORE=0 $P:USP_TSTORE=2 _variants/st128all/libusp.so _variants/st128none/libusp.so --config C3 --size 256 --rounds 5 --iters 100 2>&1 | grep variant | cut -c1-220
timeout 600 python tools/gpu/kab.py $P $P:USP_TSTORE=0 $P:USP_TSTORE=2 _variants/st128all/libusp.so _variants/st128none/libusp.so --config C4 --size 512 --rounds 3 --iters 50 2>&1 | grep variant | cut -c1-220
