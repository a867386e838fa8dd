# bench with the K_D tensor-map stores + ncu of the iteration kernels
python bench.py > gpurun_out/bench_r02_s5.json 2> gpurun_out/bench_r02_s5.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_s5.json 2> gpurun_out/bench_ref_s5.err; echo ref_rc=$?
CMD="python bench.py --steps 1 --warmup 1 --iters 3 --no-e2e --no-cpu --no-solvers --no-variants"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_s5.csv $CMD > gpurun_out/ncu_s5_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"k_xpass_pipe|k_stile" -s 10 -c 4 -o gpurun_out/prof_r02_s5_iter -f $CMD > gpurun_out/ncu_s5_full.log 2>&1; echo ncu2=$?
