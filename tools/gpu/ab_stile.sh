# A/B of the strided passes: TMA 16-column tiles (default) vs the register-staged legacy ones
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in 1 0; do
  USP_STILE=$v timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/ab_stile_$v.json 2>gpurun_out/ab_stile_$v.err
  echo "USP_STILE=$v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ab_stile_$v.json'));print(d['iteration_roofline'], d['kernel_ms_per_launch'])"
done
