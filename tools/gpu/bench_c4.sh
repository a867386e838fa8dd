timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4.json 2>gpurun_out/c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/c4.err
python -c "import json;d=json.load(open('gpurun_out/c4.json'));print(d['value'], d['roofline'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
USP_REAL=0 timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4c.json 2>gpurun_out/c4c.err; echo "c4 complex rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c4c.json'));print(d['value'], d['kernel_ms_per_launch'])"
timeout 300 python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3.json 2>gpurun_out/c3.err; echo "c3 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c3.json'));print(d['value'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
