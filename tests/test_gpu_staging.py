"""Asynchronous input staging (usp_stage_inputs): the next problem's inputs
are copied on the plan's copy stream while the current one iterates; the
staged problem gives the same result as passing its inputs directly."""
import numpy as np
import pytest

from gpu_helpers import rounded_inputs, run_gpu

pytestmark = pytest.mark.gpu


def test_staged_inputs_pipeline():
    import torch
    from paper_2207_14222_b200 import Plan
    from paper_2207_14222_b200._lib import USPError
    from synth import make

    p = make("C5", (32, 32, 64))
    med, src, dtype = rounded_inputs(p)
    src2 = np.roll(src, 5, axis=2).copy()
    ref1, _, _, _ = run_gpu(p, n_iter=25, tol=0.0)
    ref2, _, _, _ = run_gpu(p, n_iter=25, tol=0.0, med=med, src=src2, dtype=dtype)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    with pytest.raises(USPError):
        plan.set_potential("staged")                 # nothing staged yet
    hm = torch.from_numpy(med).pin_memory()
    hs1 = torch.from_numpy(src).pin_memory()
    hs2 = torch.from_numpy(src2).pin_memory()
    plan.stage_inputs(hm, hs1)
    plan.set_potential("staged")
    plan.set_source("staged")
    plan.stage_inputs(hm, hs2)                       # overlaps the iterations below
    plan.iterate(25, p.alpha, 0.0)
    x1 = plan.get_field().cpu().numpy().astype(np.complex128)
    plan.set_potential("staged")
    plan.set_source("staged")
    plan.iterate(25, p.alpha, 0.0)
    x2 = plan.get_field().cpu().numpy().astype(np.complex128)
    assert np.array_equal(x1, ref1) and np.array_equal(x2, ref2)
    with pytest.raises(USPError):
        plan.set_source("staged")                    # consumed
    # asynchronous read-back: the field lands after wait_field, even when the
    # plan stream moves on to the next problem right away
    out = torch.empty(plan.local_shape, dtype=torch.complex64).pin_memory()
    plan.get_field_async(out)
    plan.stage_inputs(hm, hs1)
    plan.set_potential("staged")
    plan.set_source("staged")
    plan.iterate(25, p.alpha, 0.0)
    plan.wait_field()
    assert np.array_equal(out.numpy().astype(np.complex128), ref2)
    plan.get_field_async(out)
    plan.wait_field()
    assert np.array_equal(out.numpy().astype(np.complex128), ref1)
