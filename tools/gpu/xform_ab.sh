nvidia-smi --query-gpu=name,clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader
P=paper_2207_14222_b200/libusp.so
timeout 900 python tools/gpu/kab.py _variants/head/libusp.so $P $P:USP_XFORM=0 --config C5 --size 1024 --rounds 3 --iters 50 2>&1 | grep variant | cut -c1-260
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader
