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


def test_staging_pairs_and_slots():
    """A staged medium is never paired with the next problem's source
    (ADVICE r1): stage_inputs refuses while the source of a taken medium is
    pending; a staging area sized without the read-back slot refuses
    get_field_async; a host pointer passed as device memory is an argument
    error, not a fault."""
    import ctypes

    import torch
    from paper_2207_14222_b200 import Plan, _lib
    from paper_2207_14222_b200._lib import USPError
    from synth import make

    p = make("C5", (32, 32, 64))
    med, src, dtype = rounded_inputs(p)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    hm = torch.from_numpy(med).pin_memory()
    hs = torch.from_numpy(src).pin_memory()
    plan.stage_inputs(hm, hs)
    plan.set_potential("staged")
    with pytest.raises(USPError) as e:
        plan.stage_inputs(hm, hs)
    assert e.value.name == "USP_ERR_STATE"
    plan.set_source("staged")
    plan.stage_inputs(hm, hs)                        # fine again
    # two-slot staging area: inputs only
    lib = plan.lib
    n2 = ctypes.c_size_t()
    _lib.check(lib.usp_staging_size(plan.handle, 0, ctypes.byref(n2)))
    n3 = ctypes.c_size_t()
    _lib.check(lib.usp_staging_size(plan.handle, 1, ctypes.byref(n3)))
    assert n3.value > n2.value
    plan2 = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    area = torch.empty(n2.value, dtype=torch.uint8, device="cuda")
    _lib.check(lib.usp_plan_set_staging(plan2.handle, ctypes.c_void_p(area.data_ptr()), n2.value))
    plan2.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan2.set_source(torch.from_numpy(src).cuda())
    out = torch.empty(plan2.local_shape, dtype=torch.complex64).pin_memory()
    assert lib.usp_get_field_async(plan2.handle, ctypes.c_void_p(out.data_ptr())) == 6   # USP_ERR_NOMEM
    # a pageable host array passed as a device pointer
    host = np.zeros(p.shape, dtype=np.complex64)
    assert lib.usp_set_source(plan2.handle, ctypes.c_void_p(host.ctypes.data), 0) == 1   # USP_ERR_ARG
    assert lib.usp_set_source(plan2.handle, ctypes.c_void_p(host.ctypes.data), 7) == 1   # bad where
    plan2.set_source(torch.from_numpy(src).cuda())   # the plan is still usable
    plan2.iterate(3, p.alpha, 0.0)


def test_real_path_async_readback():
    """usp_get_field_async on the real (float32 half-spectrum) path."""
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make("C4", (64, 64, 64))   # the real path needs y, z extents >= 64
    med, src, dtype = rounded_inputs(p)
    assert dtype == "r32"
    ref, _, _, _ = run_gpu(p, n_iter=12, tol=0.0)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    plan.stage_inputs(torch.from_numpy(med).pin_memory(), torch.from_numpy(src).pin_memory())
    plan.set_potential("staged")
    plan.set_source("staged")
    plan.iterate(12, p.alpha, 0.0)
    out = torch.empty(plan.local_shape, dtype=torch.float32).pin_memory()
    plan.get_field_async(out)
    plan.wait_field()
    assert np.array_equal(out.numpy().astype(np.complex128), ref)
    with pytest.raises(ValueError):
        plan.get_field_async(torch.empty(10, dtype=torch.float32).pin_memory())   # wrong size
