# persistent 2-D solver: CTA size variants (C2 512^2 to 1e-6), parity tests under each variant
for nt in 128 64 256 128 64; do USP_S2NT=$nt timeout 300 python tools/gpu/c2_prof.py 2>&1 | tail -1 | sed "s/^/nt=$nt /"; done
for nt in 64 128; do USP_S2NT=$nt timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "C2 or closed" 2>&1 | tail -1; done
