import sys, math, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2207_14222_b200 import Plan
shapes = [tuple(int(x) for x in s.split('x')) for s in sys.argv[1:]]
for shape in shapes:
    try:
        k0 = 2*math.pi/8; k2 = (k0*(1+0.05j))**2
        sigma, c = -k2.real, -1j*abs(k2.imag)/0.95
        plan = Plan(shape, sigma=sigma, c=c)
        plan.set_potential(torch.full(shape, k2, dtype=torch.complex64, device='cuda'), -1.0)
        S = torch.zeros(shape, dtype=torch.complex64, device='cuda'); S[tuple(s//2 for s in shape)] = 1
        plan.set_source(S)
        n, t = plan.iterate(2, 0.75, 0.0)
        print(shape, 'ok', n, plan.residual(), flush=True)
        del plan
    except Exception as e:
        print(shape, 'FAIL', e, flush=True)
        break
