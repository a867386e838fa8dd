#!/bin/bash
# ncu --set full of one K_C launch (k_stile<1024, 2>) late in a solve (dense fields), with source/SASS counters
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --iters 12 --no-e2e --no-cpu --no-solvers --no-variants"
$CMD > gpurun_out/plain_kc.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_kc.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"1024, \\(int\\)2>" -s 20 -c 1 \
    -o gpurun_out/prof_kc -f $CMD > gpurun_out/ncu_kc.log 2>&1
echo ncu_rc=$?
tail -2 gpurun_out/ncu_kc.log
