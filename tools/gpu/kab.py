"""In-process A/B of library builds on the C5 1024^3 iteration.

    python tools/gpu/kab.py LIB_A.so LIB_B.so ... [--rounds 4] [--iters 20] [--size 1024]

Each variant gets its own plan (own copy of the library: ctypes handles and
static state are per file, so copy a build to a distinct name first);
variants are run round-robin `--rounds` times so clock/thermal drift hits
them alike, and per-kernel device times (usp_profile_read) are reported as
the median over rounds.  (Builds come from tools/build_variant.py, e.g.
from another git revision of csrc/.)
"""
import argparse
import ctypes
import json
import os
import shutil
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--nz", type=int, default=None, help="planes (default: --size)")
    ap.add_argument("--opts", default="", help="plan options for every variant, e.g. flat_work=1,delta_form=1")
    args = ap.parse_args()
    popts = {k: int(v) for k, v in (o.split("=", 1) for o in args.opts.split(",") if o)}
    import torch

    from paper_2207_14222_b200 import _lib as L
    from paper_2207_14222_b200 import Plan
    from synth import make

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    p = make(args.config, (args.nz or args.size, args.size, args.size), device=str(dev))
    real = p.kind == "diffusion"   # C4: float32 data, the real (half-spectrum) path
    if real:
        med = p.medium.real.float().contiguous()
        src = p.source.real.float().contiguous()
    else:
        med = p.medium.to(torch.complex64).contiguous()
        src = p.source.to(torch.complex64).contiguous()
    del p.medium, p.source
    stream = torch.cuda.Stream(device=dev)
    plans = []
    for k, v in enumerate(args.variants):
        path, _, envs = v.partition(":")
        env = dict(e.split("=", 1) for e in envs.split(",") if e)
        lib = os.path.join("/tmp", f"kab_{k}_" + os.path.basename(path))
        shutil.copy(path, lib)
        L._lib = None
        L.LIB_PATH = lib
        for key, val in env.items():
            os.environ[key] = val
        with torch.cuda.stream(stream):
            plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev, **popts,
                        dtype="r32" if real else "c64")
        plan.set_potential(med, 0.95)
        plan.set_source(src)
        plan.iterate(3, p.alpha, 0.0)
        for key in env:
            os.environ.pop(key)
        plans.append((v, env, plan))
    res = {v: {} for v, _, _ in plans}
    for r in range(args.rounds):
        for v, env, plan in plans:
            for key, val in env.items():
                os.environ[key] = val
            plan.profile(True)
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            plan.iterate(args.iters, p.alpha, 0.0)
            eb.record(stream)
            torch.cuda.synchronize()
            prof = plan.profile_read()
            plan.profile(False)
            for key in env:
                os.environ.pop(key)
            res[v].setdefault("iter_ms_prof", []).append(ea.elapsed_time(eb) / args.iters)
            # the same without per-kernel events (events between launches
            # defeat programmatic dependent launch)
            torch.cuda.synchronize()
            ea.record(stream)
            plan.iterate(args.iters, p.alpha, 0.0)
            eb.record(stream)
            torch.cuda.synchronize()
            res[v].setdefault("iter_ms", []).append(ea.elapsed_time(eb) / args.iters)
            for name, (ms, cnt) in prof.items():   # ms per iteration (see opt_ab.py)
                if cnt:
                    res[v].setdefault(name, []).append(ms / args.iters)
    for v in res:
        out = {k: round(statistics.median(x), 4) for k, x in res[v].items()}
        out["iter_ms_all"] = [round(x, 3) for x in res[v]["iter_ms"]]
        print(json.dumps({"variant": v, **out}))


if __name__ == "__main__":
    main()
