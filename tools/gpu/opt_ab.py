"""In-process A/B of plan options (usp_plan_desc fields) on one library build.

    python tools/gpu/opt_ab.py "zpair:" "flat:flat_work=1" [--rounds 5] [--iters 20] [--config C5] [--size 1024]

Each variant is NAME:opt=val,opt=val (Plan keyword arguments); every variant
gets its own plan and workspace on the same inputs, variants run round-robin
`--rounds` times so clock / power-cap drift hits them alike, and per-kernel
device times per iteration (usp_profile_read) and the iteration time are
reported as medians over rounds, one JSON line per variant.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def _val(s):
    for f in (int, float):
        try:
            return f(s)
        except ValueError:
            pass
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--nz", type=int, default=None)
    ap.add_argument("--config", default="C5")
    args = ap.parse_args()
    import torch

    from paper_2207_14222_b200 import Plan
    from synth import make

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    p = make(args.config, (args.nz or args.size, args.size, args.size), device=str(dev))
    real = p.kind == "diffusion"
    med = (p.medium.real.float() if real else p.medium.to(torch.complex64)).contiguous()
    src = (p.source.real.float() if real else p.source.to(torch.complex64)).contiguous()
    del p.medium, p.source
    stream = torch.cuda.Stream(device=dev)
    plans = []
    for v in args.variants:
        name, _, opts = v.partition(":")
        kw = {k: _val(x) for k, x in (o.split("=", 1) for o in opts.split(",") if o)}
        with torch.cuda.stream(stream):
            plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev,
                        dtype="r32" if real else "c64", **kw)
        plan.set_potential(med, 0.95)
        plan.set_source(src)
        plan.iterate(3, p.alpha, 0.0)
        plans.append((name, kw, plan))
    res = {name: {"iter_ms": []} for name, _, _ in plans}
    for _ in range(args.rounds):
        for name, _, plan in plans:
            plan.profile(True)
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            plan.iterate(args.iters, p.alpha, 0.0)
            eb.record(stream)
            torch.cuda.synchronize()
            res[name]["iter_ms"].append(ea.elapsed_time(eb) / args.iters)
            # ms per ITERATION (an x-form plan launches one spare chain + x pass
            # per iterate() call that skips itself: per-launch averages would
            # read ~1/iters low)
            for k, (ms, n) in plan.profile_read().items():
                if n:
                    res[name].setdefault(k, []).append(ms / args.iters)
            plan.profile(False)
    for name, kw, plan in plans:
        out = {"variant": name, "options": kw, "work_layout": plan.work_layout(), "config": args.config,
               "shape": list(p.shape)}
        out.update({k: round(statistics.median(v), 4) for k, v in res[name].items()})
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
