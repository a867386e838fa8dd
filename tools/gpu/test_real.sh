timeout 900 python -m pytest tests/test_gpu_real.py -x -q 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/c4.json 2>gpurun_out/c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/c4.err
python -c "import json;d=json.load(open('gpurun_out/c4.json'));print(d['value'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
