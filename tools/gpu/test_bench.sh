# GPU suite + a short 1024^3 bench (kernel times per launch)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-solvers > gpurun_out/tb.json 2>gpurun_out/tb.err
echo "bench rc=$?"; tail -2 gpurun_out/tb.err; python -c "import json;d=json.load(open('gpurun_out/tb.json'));print(d['value'], d['config']['iteration_form'], d['roofline'], d['iteration_roofline'], d['kernel_ms_per_launch'], d['clocks'])"
