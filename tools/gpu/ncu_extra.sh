# ncu --set full of the kernels added after the first capture, each on its own small command
set -x
python tools/gpu/configs_bench.py C4 > gpurun_out/p_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_xpass_real|k_stile" -s 8 -c 2 -o gpurun_out/prof_real -f python tools/gpu/configs_bench.py C4 > gpurun_out/ncu_real.log 2>&1
python tools/gpu/c2_prof.py > gpurun_out/p_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_solve2d" -s 1 -c 1 -o gpurun_out/prof_solve2d -f python tools/gpu/c2_prof.py > gpurun_out/ncu_s2.log 2>&1
python tools/gpu/configs_bench.py C3 > gpurun_out/p_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_xop|k_kupd" -s 10 -c 5 -o gpurun_out/prof_krylov -f python tools/gpu/configs_bench.py C3 > gpurun_out/ncu_kry.log 2>&1
ls -la gpurun_out/*.ncu-rep
