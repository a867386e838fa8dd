# A/B: half-tile tensor-map stores in k_stile (USP_TSTORE=1 default) vs all-register stores
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 1 0 2; do
  USP_TSTORE=$v timeout 300 python bench.py --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu > gpurun_out/ab_ts_$v.json 2>gpurun_out/ab_ts_$v.err
  echo "USP_TSTORE=$v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ab_ts_$v.json'));print(d['iteration_roofline'], d['kernel_ms_per_launch'])"
done
