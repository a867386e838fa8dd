"""C2 (512^2, persistent 2-D solver) to 1e-6 with several library builds, round-robin."""
import os, shutil, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2207_14222_b200 import _lib as L
from paper_2207_14222_b200 import Plan
from synth import make

p = make("C2")
med = torch.from_numpy(np.asarray(p.medium).astype(np.complex64)).cuda()
src = torch.from_numpy(np.asarray(p.source).astype(np.complex64)).cuda()
plans = []
for k, path in enumerate(sys.argv[1:]):
    lib = f"/tmp/c2ab_{k}.so"
    shutil.copy(path, lib)
    L._lib = None
    L.LIB_PATH = lib
    plans.append((path, Plan(p.shape)))
res = {path: [] for path, _ in plans}
for r in range(4):
    for path, plan in plans:
        plan.set_potential(med, 0.95); plan.set_source(src)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        n, term = plan.iterate(20000, 0.75, 1e-6)
        b.record(); torch.cuda.synchronize()
        if r:
            res[path].append(a.elapsed_time(b))
        assert term == "converged", term
for path in res:
    print(path, n, "ms", sorted(res[path]))
