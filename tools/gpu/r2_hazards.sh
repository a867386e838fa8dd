timeout 1200 python -m pytest tests/test_gpu_hazards.py tests/test_gpu_staging.py -q 2>&1 | tail -15
