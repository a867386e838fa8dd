for cfg in "0 1" "1 1" "2 1" "2 0" "4 1"; do set -- $cfg
  USP_CHUNK=$1 USP_L2HINT=$2 timeout 300 python bench.py --steps 1 --warmup 3 --iters 10 --no-e2e --no-cpu --no-solvers > gpurun_out/ch.json 2>gpurun_out/ch.err
  echo "G=$1 hint=$2 rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/ch.json'));k=d['kernel_ms_per_launch']
G=int('$1') or 1024
print(round(d['iteration_roofline']['iter_ms'],3), {kk:round(v*1024/G,3) for kk,v in k.items() if kk in ('xpass','y_fwd','y_inv','z_fwd_mul_inv')}, 'per-volume-equivalent ms')"
done
