timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/tb.json 2>gpurun_out/tb.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/tb.json'));print(d['iteration_roofline'], d['kernel_ms_per_launch'], d['clocks'])"
