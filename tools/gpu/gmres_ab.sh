timeout 900 python -m pytest tests/test_gpu_krylov.py -q 2>&1 | tail -2
for v in 0 1; do USP_GMRES_CGS2=$v timeout 600 python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2207_14222_b200 import Plan
from synth import make
dev = torch.device("cuda", 0)
for name, size in (("C3", None), ("C2", None)):
    p = make(name, size, device=str(dev) if name == "C3" else None)
    import numpy as np
    med = (p.medium.to(torch.complex64) if name == "C3" else torch.from_numpy(np.asarray(p.medium).astype(np.complex64)).to(dev))
    src = (p.source.to(torch.complex64) if name == "C3" else torch.from_numpy(np.asarray(p.source).astype(np.complex64)).to(dev))
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D)
    for rep in range(2):
        plan.set_potential(med, 0.95); plan.set_source(src)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        n, term = plan.gmres(20, 20000, 1e-6)
        b.record(); torch.cuda.synchronize()
    print("CGS2=" + os.environ["USP_GMRES_CGS2"], name, n, term, round(a.elapsed_time(b), 2), "ms", flush=True)
PY
done
