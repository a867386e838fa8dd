import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2207_14222_b200 import Plan
from synth import make
def run(shape, n):
    p = make("C3", shape)
    med = np.asarray(p.medium).astype(np.complex64); src = np.asarray(p.source).astype(np.complex64)
    pl = Plan(shape, kind=p.kind, h=p.h, D=p.D)
    pl.set_potential(torch.from_numpy(med).cuda(), 0.95); pl.set_source(torch.from_numpy(src).cuda())
    out = []
    for k in n:
        pl.iterate(k, 0.75, 0.0); out.append(pl.get_field().cpu().numpy().copy())
    return out, pl.history()
shape = tuple(int(a) for a in sys.argv[1].split(","))
a, ha = run(shape, [1, 1, 5])
print("hist", ha[:8])
