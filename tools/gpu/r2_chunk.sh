timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_real.py tests/test_gpu_hazards.py -q -x 2>&1 | tail -8
python bench.py --steps 1 --warmup 1 --iters 20 --virtual-ranks 8 --separate-transposes --no-e2e --no-cpu --no-solvers --no-variants > gpurun_out/bench_sep8.json 2> gpurun_out/bench_sep8.err; echo rc=$?
tail -c 600 gpurun_out/bench_sep8.err
