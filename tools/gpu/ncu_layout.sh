#!/bin/bash
# ncu --set full of the z pass (K_C) and of one X_ITER x pass on the z-pair
# and the flat chain-buffer layouts (C5 1024^3).  K_C: iteration 2's (the
# 5th k_stile<1024,2> launch incl. the setup chain's); x pass: the 4th
# k_xpass_pipe launch (after the two setup passes and iteration 1's).
set -e
mkdir -p gpurun_out
for v in "zpair:" "flat:flat_work=1"; do
  n=${v%%:*}
  if [ "${1:-all}" != "xpass" ]; then
    ncu --set full --clock-control none -k regex:"k_stile" --launch-skip 9 --launch-count 3 \
        -o gpurun_out/ncu_layout_$n -f python tools/gpu/opt_ab.py "$v" --rounds 1 --iters 2 > gpurun_out/ncu_layout_$n.log 2>&1
  fi
  ncu --set full --clock-control none -k regex:"xpass" --launch-skip 3 --launch-count 1 \
      -o gpurun_out/ncu_layout_x_$n -f python tools/gpu/opt_ab.py "$v" --rounds 1 --iters 2 > gpurun_out/ncu_layout_x_$n.log 2>&1
done
