import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_helpers import *
from oracle import oracle as O
from synth import make
O.build()
for name, shape, n, tol in [('C1', None, 2000, 1e-6), ('C5', (32,32,32), 20, 0.0), ('C2', (64,64), 50, 0.0)]:
    p = make(name, shape)
    t = time.time()
    xg, ng, term, plan = run_gpu(p, n_iter=n, tol=tol)
    t1 = time.time()
    res, sp = run_oracle(O, p, n_iter=n, tol=tol)
    ref, _ = run_oracle(O, p, n_iter=ng, tol=0.0)
    print(name, shape, 'gpu n', ng, term, 'oracle n', res.n_done, 'relL2', rel_l2(xg, ref.x), 'split', plan.split, 'hist', plan.history()[:4], res.hist[:4], 'gpu t', t1-t, flush=True)
