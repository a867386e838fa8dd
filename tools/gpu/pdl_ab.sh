P=paper_2207_14222_b200/libusp.so
timeout 600 python tools/gpu/kab.py $P $P:USP_PDL=0 --config C3 --size 256 --rounds 5 --iters 100 2>&1 | grep variant | cut -c1-200
timeout 600 python tools/gpu/kab.py $P $P:USP_PDL=0 --config C4 --size 512 --rounds 5 --iters 50 2>&1 | grep variant | cut -c1-200
timeout 600 python tools/gpu/kab.py $P $P:USP_PDL=0 --config C5 --size 1024 --rounds 3 --iters 10 2>&1 | grep variant | cut -c1-200
