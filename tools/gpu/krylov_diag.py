import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from oracle import oracle as O
from synth import make
from test_gpu_krylov import _gpu, _orc
from gpu_helpers import rel_l2
O.build()
for name, shape in [("C2", (128, 128)), ("C3", (64, 64, 64)), ("C2", (512, 512))]:
    p = make(name, shape)
    for n in (2, 5, 10, 20, 40):
        x, nd, term, plan = _gpu(p, n, 0.0)
        ref = _orc(O, p, n, 0.0)
        print(name, shape, n, "relL2 %.2e" % rel_l2(x, ref.x), "gpu r %.3e oracle r %.3e" % (plan.history()[n], ref.hist[2*n-1]), flush=True)
    for tol in (1e-4, 1e-5, 1e-6):
        x, nd, term, plan = _gpu(p, 3000, tol)
        ref = _orc(O, p, 3000, tol)
        print(name, shape, "tol", tol, "gpu", nd, term, "oracle", ref.n_done, ref.half, "relL2 %.2e" % rel_l2(x, ref.x), flush=True)
