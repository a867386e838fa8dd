#!/bin/bash
# antisymmetrised / tensor-diffusion capability kernels: parity tests, hazards, timings, ncu
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tdiff.py tests/test_gpu_anti.py tests/test_gpu_hazards.py -x -q > gpurun_out/anti_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/anti_tests.log
timeout 600 python tools/gpu/capability_runs.py > gpurun_out/capability_anti.log 2>&1; echo "cap rc=$?" >> gpurun_out/capability_anti.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_tdiff|k_xfft|k_stile" -c 60 --csv python tools/gpu/capability_runs.py --only tdiff > gpurun_out/ncu_tdiff.csv 2> gpurun_out/ncu_tdiff.err
tail -3 gpurun_out/anti_tests.log
