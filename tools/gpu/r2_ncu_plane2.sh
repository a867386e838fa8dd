cp paper_2207_14222_b200/libusp.so /tmp/libusp_ncu.so
CMD="python tools/gpu/kab.py /tmp/libusp_ncu.so --nz 256 --iters 2 --rounds 1"
$CMD > gpurun_out/ncu_plane2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_plane -s 4 -c 1 -o gpurun_out/prof_plane2 $CMD > gpurun_out/ncu_plane2.log 2>&1
echo rc=$?
