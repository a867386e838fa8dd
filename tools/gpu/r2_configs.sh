timeout 600 python -m pytest tests/test_gpu_hazards.py -q -k "plane" 2>&1 | tail -3
timeout 1200 python tools/gpu/configs_bench.py C1 C2 C3 C4 C5 > gpurun_out/configs_r02.jsonl 2> gpurun_out/configs_r02.err; echo rc=$?
