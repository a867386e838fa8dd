python -m pytest tests/test_gpu_krylov.py tests/test_gpu_hazards.py -q > gpurun_out/kr.log 2>&1; tail -5 gpurun_out/kr.log
