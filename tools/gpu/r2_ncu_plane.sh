CMD="python bench.py --steps 1 --warmup 1 --iters 4 --no-e2e --no-cpu --no-solvers --no-variants"
$CMD > gpurun_out/ncu_plane_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_plane -s 3 -c 1 -o gpurun_out/prof_plane $CMD > gpurun_out/ncu_plane.log 2>&1
echo rc=$?
