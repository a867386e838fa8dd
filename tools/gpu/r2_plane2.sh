timeout 900 python -m pytest tests/test_gpu_plane.py -x -q 2>&1 | tail -15
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-solvers > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?
tail -c 1500 gpurun_out/bench2.err
