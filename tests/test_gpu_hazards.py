"""Hazard checks without compute-sanitizer (closed on this GPU pool: runs
under it have left GPUs needing a reset; profiles/sanitizer_r02.txt).

* Determinism: every kernel family runs the same solve twice in one process;
  the fields and residual histories must be bit-identical.  The library's
  reductions are fixed-order by design, so any difference is a race (a read
  before the matching write, a stage reused too early, a missed barrier).
* Poisoned workspace: the caller-owned workspace is filled with NaN bytes
  before the solve; the result must equal the one from a zero-filled
  workspace bit for bit -- a read of workspace memory the library never
  wrote (an uninitialised-read hazard) would propagate a NaN or change bits.
"""
import numpy as np
import pytest

from gpu_helpers import rounded_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


CASES = [
    ("C3", (32, 32, 32), 400, 1e-6, {}),                       # x-form, sparse source, switch, stop
    ("C5", (32, 64, 128), 12, 0.0, {"delta_form": True}),      # Delta-form, ragged 3-D
    ("C5", (32, 64, 128), 12, 0.0, {"dense_source": True}),    # dense x-form
    ("C2", (64, 64), 60, 0.0, {}),                             # persistent 2-D solver, grid barrier
    ("C2", (64, 64), 20, 0.0, {"launch_per_pass": True}),
    ("C1", None, 60, 0.0, {}),                                 # 1-D on-chip solve
    ("C5", (64, 64, 32), 8, 0.0, {"virtual_ranks": 2}),        # fused peer-store transposes
    ("C5", (64, 64, 32), 8, 0.0, {"virtual_ranks": 4, "separate_transposes": True}),
    ("C4", (64, 64, 64), 30, 0.0, {}),                         # real path across the form switch
    ("C5", (1024, 64, 16), 3, 0.0, {}),                        # k_stile<1024> two-round exchange, TMA stores,
                                                               # z pass on the plane-pair buffer
    ("C5", (1024, 64, 16), 3, 0.0, {"flat_work": True}),       # the same z pass in place on work
    ("C3", (128, 64, 256), 6, 0.0, {"delta_form": True}),      # plane-pair buffer, full exchange (N = 128)
    ("C5", (64, 1024, 1024), 4, 0.0, {"plane_chain": True}),   # plane-chained pass
    ("C5", (64, 64, 64), 5, 0.0, {"antisymmetric": True}),
    ("C5", (64, 64, 1024), 3, 0.0, {"antisymmetric": True}),  # k_anti_pipe<1024>, 3 stages
]


def _refill(plan, fill):
    """Fill the workspace and hand it over again (usp_plan_set_workspace
    initialises what the library needs initialised, e.g. the real path's
    spectrum padding)."""
    import ctypes

    import torch
    from paper_2207_14222_b200 import _lib

    plan.workspace.fill_(fill)
    torch.cuda.synchronize()
    _lib.check(plan.lib.usp_plan_set_workspace(plan.handle, ctypes.c_void_p(plan.workspace.data_ptr()),
                                               plan.workspace.numel()))


def _solve(name, shape, n, tol, opts, fill=None):
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make(name, shape)
    med, src, dtype = rounded_inputs(p)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, **opts)
    if fill is not None:
        _refill(plan, fill)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.from_numpy(src).cuda())
    nd, term = plan.iterate(n, p.alpha, tol)
    x = plan.get_field().cpu().numpy()
    h = plan.history()
    plan.close()
    return x, nd, term, h


@pytest.mark.parametrize("name,shape,n,tol,opts", CASES)
def test_repeat_is_bit_identical(name, shape, n, tol, opts):
    a = _solve(name, shape, n, tol, opts)
    b = _solve(name, shape, n, tol, opts)
    assert a[1] == b[1] and a[2] == b[2]
    assert np.array_equal(a[0].view(np.uint8), b[0].view(np.uint8))
    assert np.array_equal(a[3], b[3])


@pytest.mark.parametrize("name,shape,n,tol,opts", CASES)
def test_poisoned_workspace(name, shape, n, tol, opts):
    z = _solve(name, shape, n, tol, opts, fill=0)
    q = _solve(name, shape, n, tol, opts, fill=255)      # 0xFF bytes: NaN in every float32 / float64
    assert np.isfinite(q[0]).all()
    assert np.array_equal(z[0].view(np.uint8), q[0].view(np.uint8))
    assert np.array_equal(z[3], q[3])


def test_krylov_repeat_and_poison():
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make("C5", (32, 32, 64))
    med, src, _ = rounded_inputs(p)
    outs = []
    for fill in (0, 255, 0):
        plan = Plan(p.shape)
        _refill(plan, fill)
        plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
        plan.set_source(torch.from_numpy(src).cuda())
        plan.bicgstab(1, 0.0)                    # allocates the Krylov workspace
        plan.kworkspace.fill_(fill)
        plan.set_source(torch.from_numpy(src).cuda())
        nb, _ = plan.bicgstab(6, 0.0)
        xb = plan.get_field().cpu().numpy()
        plan.set_source(torch.from_numpy(src).cuda())
        plan.gmres(5, 1, 0.0)
        plan.gworkspace.fill_(fill)
        plan.set_source(torch.from_numpy(src).cuda())
        ng, _ = plan.gmres(5, 12, 0.0)
        xg = plan.get_field().cpu().numpy()
        outs.append((xb, xg))
        plan.close()
    for xb, xg in outs[1:]:
        assert np.array_equal(xb.view(np.uint8), outs[0][0].view(np.uint8))
        assert np.array_equal(xg.view(np.uint8), outs[0][1].view(np.uint8))


@pytest.mark.parametrize("shape", [(64, 64, 128), (64, 512)])
def test_tdiff_repeat_and_poison(shape):
    """Tensor diffusion: the fused pipelined x pass (3-D) and its 2-D
    two-stage instance, zero / NaN / zero workspace: bit-identical."""
    import torch
    from paper_2207_14222_b200 import Plan

    rng = np.random.default_rng(12)
    d = len(shape)
    mu = (0.02 + 0.08 * rng.random(shape)).astype(np.float32)
    A = rng.standard_normal(shape + (d, d)) * 0.3
    D = (np.einsum("...ij,...kj->...ik", A, A) + np.eye(d)).astype(np.float32)
    S = np.zeros(shape, dtype=np.float32)
    S[tuple(s // 2 for s in shape)] = 1.0
    outs = []
    for fill in (0, 255, 0):
        plan = Plan(shape, kind="diffusion", tensor_diffusion=True)
        _refill(plan, fill)
        plan.set_tensor_medium(torch.from_numpy(mu).cuda(), torch.from_numpy(D).cuda(), 0.95)
        plan.set_source(torch.from_numpy(S).cuda())
        plan.iterate(12, 0.75, 0.0)
        outs.append((plan.get_field().cpu().numpy(), plan.history()[:13].copy()))
        plan.close()
    assert np.isfinite(outs[1][0]).all()
    for u, h in outs[1:]:
        assert np.array_equal(u.view(np.uint8), outs[0][0].view(np.uint8))
        assert np.array_equal(h, outs[0][1])
