timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for g in 0 4 8 16; do
  USP_CHUNK=$g timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/ch$g.json 2>gpurun_out/ch$g.err
  echo "G=$g rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ch$g.json'));print(round(d['value']/1e9,2), d['iteration_roofline'], d['roofline']['frac'], d['kernel_ms_per_launch'])"
done
