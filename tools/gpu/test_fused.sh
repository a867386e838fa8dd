timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_real.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for P in 2 8; do
timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu --virtual-ranks $P > gpurun_out/bf$P.json 2>gpurun_out/bf$P.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bf$P.json'));print(d['value'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
done
