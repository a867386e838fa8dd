import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2207_14222_b200 import Plan
from synth import make
p = make("C2")
med = torch.from_numpy(np.asarray(p.medium).astype(np.complex64)).cuda()
src = torch.from_numpy(np.asarray(p.source).astype(np.complex64)).cuda()
plan = Plan(p.shape)
for rep in range(2):
    plan.set_potential(med, 0.95); plan.set_source(src)
    plan.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    n, term = plan.iterate(2000, 0.75, 1e-6)
    b.record(); torch.cuda.synchronize()
    prof = plan.profile_read(); plan.profile(False)
    print(n, term, a.elapsed_time(b), {k: (round(v[0], 3), v[1], round(v[0] / v[1] * 1e3, 2)) for k, v in prof.items()})
# without profiling events
plan.set_potential(med, 0.95); plan.set_source(src)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
n, term = plan.iterate(2000, 0.75, 1e-6)
b.record(); torch.cuda.synchronize()
print("no-prof", n, a.elapsed_time(b))
