timeout 900 python bench.py --virtual-ranks 8 --steps 2 --warmup 3 --no-e2e --no-cpu --no-solvers > gpurun_out/virt8.json 2> gpurun_out/virt8.err; echo "virt rc=$?"; tail -1 gpurun_out/virt8.err
python -c "import json;d=json.load(open('gpurun_out/virt8.json'));print(d['value'], d['config']['parallelism'], d['config']['iteration_form'], d['iteration_roofline'], d['kernel_ms_per_launch'])"
timeout 1200 python tools/gpu/configs_bench.py C1 C2 C3 C4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
