timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "0 1" "4 1" "8 1" "8 0" "16 1"; do set -- $cfg
  USP_CHUNK=$1 USP_L2HINT=$2 timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/ch.json 2>gpurun_out/ch.err
  echo "G=$1 hint=$2 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ch.json'));print(round(d['value']/1e9,2), round(d['iteration_roofline']['iter_ms'],3), {k:round(v,4) for k,v in d['kernel_ms_per_launch'].items()})"
done
