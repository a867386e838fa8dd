#!/bin/bash
# setup kernels (k_potential, k_farthest) after the one-wave grid clamp: parity tests + a short bench
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_staging.py tests/test_gpu_real.py -q -x > gpurun_out/setup_tests.log 2>&1; tail -3 gpurun_out/setup_tests.log
python bench.py --steps 3 --warmup 3 --no-variants --no-solvers --no-cpu > gpurun_out/bench_setup.json 2> gpurun_out/bench_setup.err; echo bench_rc=$?
