#!/bin/bash
# capability paths (antisymmetrised, tensor diffusion, BiCGSTAB, GMRES): their GPU tests, device timings, ncu metrics
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tdiff.py tests/test_gpu_anti.py tests/test_gpu_krylov.py tests/test_gpu_hazards.py -x -q > gpurun_out/cap_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cap_tests.log
timeout 600 python tools/gpu/capability_runs.py > gpurun_out/capability.log 2>&1; echo "cap rc=$?" >> gpurun_out/capability.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gs|k_kupd|k_xop|k_anti|k_tdiff|k_stile|k_xfft" --csv python tools/gpu/capability_runs.py > gpurun_out/ncu_capability.csv 2> gpurun_out/ncu_capability.err
tail -3 gpurun_out/cap_tests.log
