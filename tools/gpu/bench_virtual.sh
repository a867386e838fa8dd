timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/bv1.json 2>gpurun_out/bv1.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bv1.json'));print(d['value'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
for P in 2 8; do
timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu --virtual-ranks $P > gpurun_out/bv$P.json 2>gpurun_out/bv$P.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bv$P.json'));print(d['value'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
done
tail -3 gpurun_out/bv2.err
