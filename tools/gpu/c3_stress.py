"""C3 256^3 to 1e-6 repeated: history monotone? identical across runs?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2207_14222_b200 import Plan
from synth import make

p = make("C3", device="cuda")
med, src = p.medium.to(torch.complex64), p.source.to(torch.complex64)
ref = None
for rep in range(12):
    plan = Plan(p.shape)
    plan.set_potential(med, 0.95)
    plan.set_source(src)
    n, term = plan.iterate(500, 0.75, 1e-6)
    h = plan.history()
    x = plan.get_field()
    d = np.diff(h[: n + 1])
    bad = np.nonzero(d > 1e-5 * h[:n])[0]
    same = None
    if ref is None:
        ref = (h.copy(), x.clone())
    else:
        same = (np.array_equal(h, ref[0]), bool(torch.equal(x, ref[1])))
    print(rep, n, term, len(h), "violations:", [(int(i), float(h[i]), float(h[i + 1])) for i in bad[:5]], "same as first:", same, flush=True)
    plan.close()
    del plan
    # churn the allocator like a test suite does
    junk = [torch.empty(int(2**27 * (1 + (rep % 3))), dtype=torch.uint8, device="cuda") for _ in range(3)]
    del junk
