"""GPU tests of the slab decomposition (include/usp.h):
the multi-GPU path's kernels, layouts and index arithmetic run on one GPU in
virtual mode (P slabs, transposes as device copies).

* Every per-element operation of the decomposed path is the same as on one
  slab (same line FFTs, same multiplier inputs, same reduction tree), so the
  field is BIT-IDENTICAL to the P = 1 path -- the strongest check of the
  send / receive layouts and the 5-D tensor-map reads.
* It also matches the oracle (relative L2 <= 1e-4) and the closed form for
  constant V on ragged grids.
"""
import math

import numpy as np
import pytest

from gpu_helpers import TOL_FIELD, rel_l2, rounded_inputs, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _run(p, n, virtual_ranks, tol=0.0, **opts):
    import torch
    from paper_2207_14222_b200 import Plan

    med, src, dtype = rounded_inputs(p)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, virtual_ranks=virtual_ranks, **opts)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.from_numpy(src).cuda())
    nd, term = plan.iterate(n, p.alpha, tol)
    return plan.get_field().cpu().numpy(), nd, term, plan


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("name,shape,P,n", [("C3", (64, 64, 64), 2, 40), ("C3", (128, 64, 64), 4, 30),
                                            ("C5", (64, 128, 64), 8, 20), ("C4", (64, 64, 128), 2, 30),
                                            ("C3", (256, 128, 64), 2, 10), ("C3", (64, 64, 64), 16, 10),
                                            ("C5", (2048, 64, 32), 8, 6)])
def test_virtual_slabs_bit_identical_to_one_slab(name, shape, P, n, fused):
    """fused = transposes in the K_B / K_C stores (peer-memory path; P <= 8);
    0 = separate transposes (device copies standing in for the NCCL
    all-to-alls)."""
    from synth import make

    p = make(name, shape)
    x1, n1, _, pl1 = _run(p, n, 0)
    xp, n_p, _, plp = _run(p, n, P, separate_transposes=fused == "0")
    assert n1 == n_p == n
    assert plp.local_shape == tuple(shape) and plp.z0 == 0
    assert np.array_equal(x1.view(np.uint8), xp.view(np.uint8)), rel_l2(xp.astype(np.complex128), x1.astype(np.complex128))
    assert np.array_equal(pl1.history(), plp.history())
    s1, sp = pl1.split, plp.split
    assert s1.c == sp.c and s1.sigma == sp.sigma


@pytest.mark.parametrize("name,shape,P,n", [("C3", (64, 64, 64), 4, 120), ("C4", (64, 64, 64), 2, 100)])
def test_virtual_slabs_match_oracle(orc, name, shape, P, n):
    from synth import make

    p = make(name, shape)
    xg, nd, term, plan = _run(p, n, P)
    assert nd == n and term == "max_iter"
    res, _ = run_oracle(orc, p, n_iter=n)
    err = rel_l2(xg.astype(np.complex128), res.x)
    assert err <= TOL_FIELD, err
    assert np.allclose(plan.history()[:n], res.hist[:n], rtol=1e-3, atol=0.0)


def test_virtual_slabs_converge_like_oracle(orc):
    """Tolerance run: same stop decision (iteration count within +-1)."""
    from synth import make

    p = make("C3", (64, 64, 64))
    xg, nd, term, plan = _run(p, 500, 4, tol=1e-6)
    res, _ = run_oracle(orc, p, n_iter=500, tol=1e-6)
    assert term == "converged" and abs(nd - res.n_done) <= 1, (nd, res.n_done)


@pytest.mark.parametrize("shape,P", [((64, 64, 64), 2), ((64, 128, 256), 4), ((128, 64, 64), 8)])
def test_virtual_slabs_closed_form(shape, P):
    """Constant V: x^_k = x^*(1 - q^k) per Fourier mode (as in
    test_gpu_parity.test_closed_form_constant_V) through the decomposed path."""
    import torch
    from paper_2207_14222_b200 import Plan

    k0, nn = 2 * math.pi / 8, 1.0 + 0.05j
    k2 = (k0 * nn) ** 2
    sigma, c = -k2.real, -1j * abs(k2.imag) / 0.95
    alpha, D = 0.75, 1.0
    S = np.zeros(shape, dtype=np.complex64)
    S[tuple(s // 3 for s in shape)] = 1.0
    S[tuple(s // 5 for s in shape)] = 0.5 - 0.25j
    plan = Plan(shape, sigma=sigma, c=c, virtual_ranks=P)
    plan.set_potential(torch.full(shape, k2, dtype=torch.complex64, device="cuda"), -1.0)
    plan.set_source(torch.from_numpy(S).cuda())
    w = -complex(np.complex64(k2))
    b = 1.0 - (w - sigma) / c
    p2 = sum(np.meshgrid(*[(2 * np.pi * np.fft.fftfreq(n)) ** 2 for n in shape], indexing="ij"))
    ghat = c / (D * p2 + sigma + c)
    q = 1.0 - alpha * b * (1.0 - b * ghat)
    xstar = ghat * np.fft.fftn(S.astype(np.complex128) / c) / (1.0 - b * ghat)
    k = 12
    n, _ = plan.iterate(k, alpha, 0.0)
    x = plan.get_field().cpu().numpy().astype(np.complex128)
    err = rel_l2(x, np.fft.ifftn(xstar * (1.0 - q ** k)))
    assert n == k and err <= 2e-5, err


def test_slab_decomposition_rejects_bad_layouts():
    from paper_2207_14222_b200 import Plan, USPError

    with pytest.raises(USPError, match="UNSUPPORTED"):
        Plan((64, 64), virtual_ranks=2)                       # 2-D
    with pytest.raises(USPError, match="UNSUPPORTED"):
        Plan((64, 64, 64), virtual_ranks=3)                   # not a power of two
    with pytest.raises(USPError, match="UNSUPPORTED"):
        Plan((32, 64, 64), virtual_ranks=2)                   # nz outside the TMA-tiled range [64, 2048]
    with pytest.raises(USPError, match="UNSUPPORTED"):
        Plan((64, 64, 64), virtual_ranks=128)                 # P does not divide


def test_nccl_communicator_single_rank():
    """The run-time NCCL shim: unique id, communicator of one rank, and a
    plan on it (P = 1: no transposes) give the single-GPU result."""
    import os

    import torch
    import torch.distributed as dist
    from paper_2207_14222_b200 import Plan, comm_init
    from synth import make

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29731")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = comm_init()
        assert comm.nranks == 1 and comm.rank == 0
        p = make("C3", (64, 64, 64))
        med, src, _ = rounded_inputs(p)
        plan = Plan(p.shape, comm=comm)
        plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
        plan.set_source(torch.from_numpy(src).cuda())
        plan.iterate(10, p.alpha, 0.0)
        x = plan.get_field().cpu().numpy()
        x1, _, _, _ = _run(p, 10, 0)
        assert np.array_equal(x, x1)
        plan.close()
        comm.close()
    finally:
        if own:
            dist.destroy_process_group()


def test_rank_finish_path_with_xform_switch(monkeypatch):
    """The rank-ordered finish (x pass total -> NCCL all-gather -> k_finish)
    that P > 1 ranks use, forced on a one-rank communicator: the x-form
    passes, the switch to the Delta-form, the pending stop and the probe of a
    residual query give the single-GPU result bit for bit (reading R-30)."""
    import os

    import torch
    import torch.distributed as dist
    from paper_2207_14222_b200 import Plan, comm_init
    from synth import make

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29733")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        p = make("C3", (64, 64, 64))
        med, src, _ = rounded_inputs(p)
        x1, n1, t1, pl1 = _run(p, 2000, 0, tol=1e-6)
        comm = comm_init()
        plan = Plan(p.shape, comm=comm, test_hooks=1)   # USP_HOOK_RANK_FINISH
        plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
        plan.set_source(torch.from_numpy(src).cuda())
        n, term = plan.iterate(7, p.alpha, 0.0)
        r7 = plan.residual()                       # probe pass through k_finish
        n2, term = plan.iterate(2000, p.alpha, 1e-6)
        x = plan.get_field().cpu().numpy()
        assert plan.launch_count() > 0 and term == t1 == "converged"
        assert n + n2 == n1
        assert np.array_equal(x, x1)
        assert np.array_equal(plan.history(), pl1.history())
        assert r7[2] == 7 and r7[0] == pl1.history()[7]
        plan.close()
        comm.close()
    finally:
        if own:
            dist.destroy_process_group()


def test_nccl_window_machinery_one_rank():
    """NEXT-1's transport on one GPU: the workspace of a
    communicator plan comes from usp_shared_alloc (ncclMemAlloc), is
    registered as an NCCL 2.28 window (ncclCommWindowRegister), and values
    written through ncclGetPeerPointer's mapping of rank 0 read back through
    the plain pointer, and the device communicator's LSA barrier (the fused
    transposes' cross-rank barrier) runs (USP_HOOK_WINDOW); the solve on that
    memory is the single-GPU one bit for bit."""
    import os

    import torch
    import torch.distributed as dist
    from paper_2207_14222_b200 import Plan, comm_init
    from synth import make

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29734")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        p = make("C3", (64, 64, 128))
        med, src, _ = rounded_inputs(p)
        x1, n1, t1, pl1 = _run(p, 30, 0)
        assert pl1.transport() == "none"
        comm = comm_init()
        plan = Plan(p.shape, comm=comm, test_hooks=2)   # USP_HOOK_WINDOW
        assert plan.transport() == "nccl-window"
        plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
        plan.set_source(torch.from_numpy(src).cuda())
        n, term = plan.iterate(30, p.alpha, 0.0)
        assert n == n1 == 30
        assert np.array_equal(plan.get_field().cpu().numpy(), x1)
        plan.close()
        comm.close()
    finally:
        if own:
            dist.destroy_process_group()


def test_transport_reported():
    """usp_transport: the mode the transposes run in."""
    from synth import make

    p = make("C3", (64, 64, 64))
    assert _run(p, 2, 2)[3].transport() == "virtual"
    assert _run(p, 2, 2, separate_transposes=True)[3].transport() == "virtual-copy"
    assert _run(p, 2, 0)[3].transport() == "none"
