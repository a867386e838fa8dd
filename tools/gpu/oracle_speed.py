"""Oracle throughput on the GPU box's host cores (C3 recipe at 256^3 and the
C4 recipe at 512^3): voxel-iterations/s of orc_fixed_point."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle as O
from synth import make

O.build()
print("threads", O.num_threads(), flush=True)
for name, shape, n in (("C3", (256, 256, 256), 4), ("C4", (512, 512, 512), 2)):
    t0 = time.time()
    p = make(name, shape, device="cuda")
    med = p.medium.cpu().numpy().astype(np.complex128)
    src = p.source.cpu().numpy().astype(np.complex128)
    t1 = time.time()
    sp = O.canonical(p.kind, med, 0.95, D=p.D)
    w = O.medium_to_w(p.kind, med)
    t2 = time.time()
    res = O.fixed_point(w, src, p.h, sp.D, sp.sigma, sp.c, 0.75, 0.0, n)
    t3 = time.time()
    nv = int(np.prod(shape))
    print(f"{name} {shape}: synth {t1-t0:.1f}s canonical {t2-t1:.1f}s fixed_point({n}) {t3-t2:.1f}s "
          f"-> {nv*n/(t3-t2):.3e} vox-it/s (incl. setup round trip)", flush=True)
