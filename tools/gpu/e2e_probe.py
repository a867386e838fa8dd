"""Where the end-to-end step time goes (C5, staged inputs + async read-back)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2207_14222_b200 import Plan
from synth import make

dev = torch.device("cuda", 0)
p = make("C5", None, device=str(dev))
stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev)
h_med = torch.empty(plan.local_shape, dtype=torch.complex64, pin_memory=True)
h_src = torch.empty(plan.local_shape, dtype=torch.complex64, pin_memory=True)
h_med.copy_(p.medium.to(torch.complex64)); h_src.copy_(p.source.to(torch.complex64))
del p.medium, p.source
torch.cuda.empty_cache()
h_out = torch.empty_like(h_med).pin_memory()
t = time.perf_counter()
def lap(name):   # host wall time of each call (no device-wide syncs: the overlap is real)
    global t
    now = time.perf_counter(); print(f"{name:28s} {1e3 * (now - t):8.1f} ms", flush=True); t = now
plan.stage_inputs(h_med, h_src); lap("stage (not waited)")
for k in range(3):
    plan.set_potential("staged", 0.95); lap(f"[{k}] set_potential(staged)")
    plan.set_source("staged"); lap(f"[{k}] set_source(staged)")
    plan.stage_inputs(h_med, h_src); lap(f"[{k}] stage next (call)")
    plan.iterate(100, 0.75, 0.0); lap(f"[{k}] iterate 100")
    plan.get_field_async(h_out); lap(f"[{k}] get_field_async (call)")
plan.wait_field(); lap("wait_field")
torch.cuda.synchronize(); lap("device idle")
