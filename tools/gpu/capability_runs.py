"""A few iterations of each capability path at a real size, for an ncu
metrics pass (DRAM bytes and time per kernel -> achieved bandwidth):
antisymmetrised system (256^3), first-order tensor diffusion (3-D 256^3),
BiCGSTAB and GMRES(20) on C3 (256^3), the persistent 2-D solver (C2 512^2),
the 1-D solver (C1).  Also prints device times per path (CUDA events)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2207_14222_b200 import Plan  # noqa: E402
from synth import make  # noqa: E402


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    torch.cuda.set_device(0)
    res = {}
    if only == "tdiff":
        tdiff(res)
        print(json.dumps(res), flush=True)
        return
    # antisymmetrised system (Eq. 9-10) on the C3 recipe at 256^3
    p = make("C3", device="cuda")
    med, src = p.medium.to(torch.complex64), p.source.to(torch.complex64)
    plan = Plan(p.shape, antisymmetric=True)
    plan.set_potential(med, 0.95)
    plan.set_source(src)
    plan.iterate(2, 0.75, 0.0)
    ms, _ = timed(lambda: plan.iterate(10, 0.75, 0.0))
    res["anti_256^3"] = {"ms_per_iteration": ms / 10}
    plan.close()
    # BiCGSTAB and GMRES(20) on C3
    plan = Plan(p.shape)
    for solver in ("bicgstab", "gmres20"):
        plan.set_potential(med, 0.95)
        plan.set_source(src)
        if solver == "bicgstab":
            plan.bicgstab(2, 0.0)
            plan.set_source(src)
            ms, _ = timed(lambda: plan.bicgstab(10, 0.0))
            res["bicgstab_C3"] = {"ms_per_pass": ms / 10}
        else:
            plan.gmres(20, 2, 0.0)
            plan.set_source(src)
            ms, _ = timed(lambda: plan.gmres(20, 20, 0.0))
            res["gmres20_C3"] = {"ms_per_step": ms / 20}
    plan.close()
    del med, src
    torch.cuda.empty_cache()
    tdiff(res)
    # C2 persistent 2-D solver and C1 1-D solver
    for name in ("C2", "C1"):
        q = make(name)
        m2, s2 = (torch.from_numpy(np.asarray(q.medium).astype(np.complex64)).cuda(),
                  torch.from_numpy(np.asarray(q.source).astype(np.complex64)).cuda())
        plan = Plan(q.shape)
        plan.set_potential(m2, 0.95)
        plan.set_source(s2)
        plan.iterate(5, 0.75, 0.0)
        ms, _ = timed(lambda: plan.iterate(200, 0.75, 0.0))
        res[name] = {"ms_per_iteration": ms / 200}
        plan.close()
    print(json.dumps(res), flush=True)


def tdiff(res):
    """tensor diffusion, 3-D 256^3, anisotropic D"""
    shape = (256, 256, 256)
    rng = np.random.default_rng(3)
    mu = torch.from_numpy((0.02 + 0.08 * rng.random(shape)).astype(np.float32)).cuda()
    D = torch.zeros(shape + (3, 3), dtype=torch.float32, device="cuda")
    for i in range(3):
        D[..., i, i] = 1.0 + 0.5 * i
    D[..., 0, 1] = D[..., 1, 0] = 0.2
    S = torch.zeros(shape, dtype=torch.float32, device="cuda")
    S[128, 128, 128] = 1.0
    plan = Plan(shape, kind="diffusion", tensor_diffusion=True)
    plan.set_tensor_medium(mu, D, 0.95)
    plan.set_source(S)
    plan.iterate(2, 0.75, 0.0)
    ms, _ = timed(lambda: plan.iterate(10, 0.75, 0.0))
    res["tdiff_256^3"] = {"ms_per_iteration": ms / 10}
    plan.close()
    del mu, D, S
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
