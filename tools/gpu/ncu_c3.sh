#!/bin/bash
# ncu --set full of C3 (256^3) iteration kernels: one x pass (x-form, sparse
# source) and one z pass, to see why the x pass runs at ~63 % of the copy
# peak at this size (97 % at 1024^3)
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:"xpass|k_stile" --launch-skip 9 --launch-count 4 \
    -o gpurun_out/ncu_c3 -f python tools/gpu/opt_ab.py "v:" --config C3 --size 256 --rounds 1 --iters 3 > gpurun_out/ncu_c3.log 2>&1
echo ncu_rc=$?
