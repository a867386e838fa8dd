# ncu --set full of one iteration's strided passes (y fwd, z fwd*mul*inv, y inv) at 1024^3
set -e
CMD="python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_strided -s 3 -c 3 \
    -o gpurun_out/prof_strided -f $CMD > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
