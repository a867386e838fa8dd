"""Probe: per-kernel throughput when a pass's `work` array is L2-resident.

Runs the 4-pass iteration on (nz, ny, 1024) grids whose work array (written
by K_D, read by K_A) is 32 MB .. 8 GB, i.e. from well inside the 126 MB L2
to the full 1024^3 grid, and prints each
kernel's Gvoxel/s.  If K_A / K_B / K_D run faster per voxel on the small
grids, a persistent plane-chained schedule (K_D -> K_A -> K_B per plane,
72 instead of 104 HBM B/voxel) can pay; if not, they are not HBM-bound there.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2207_14222_b200 import Plan  # noqa: E402

res = []
for spec in (sys.argv[1:] or ["16x256", "16x512", "16x1024", "64x1024", "1024x1024"]):
    nz, ny = (int(t) for t in spec.split("x"))
    shape = (nz, ny, 1024)
    plan = Plan(shape, kind="helmholtz")
    g = torch.Generator(device="cuda").manual_seed(1)
    k0 = 2 * np.pi / 8
    n = 1.33 + 0.12 * torch.rand(shape, device="cuda", generator=g)
    med = ((k0 * n) ** 2).to(torch.complex64) + 0.05j
    plan.set_potential(med, 0.95)
    src = torch.zeros(shape, dtype=torch.complex64, device="cuda")
    src[nz // 2, ny // 2, 512] = 1
    plan.set_source(src)
    iters = max(20, min(2000, 20 * 1024 * 1024 // (nz * ny)))
    plan.iterate(10, 0.75, 0.0)
    torch.cuda.synchronize()
    plan.profile(True)
    plan.iterate(iters, 0.75, 0.0)
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    vox = nz * ny * 1024
    row = {"nz": nz, "ny": ny, "work_MB": vox * 8 >> 20, "iters": iters}
    for k, (ms, cnt) in prof.items():
        if cnt:
            row[k] = round(vox / (ms / cnt) / 1e6, 2)   # Gvoxel/s per launch
    res.append(row)
    print(json.dumps(row), flush=True)
    plan.close()
    del med, src, n
    torch.cuda.empty_cache()
