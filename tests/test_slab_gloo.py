"""world_size 2 and 4 gloo runs on CPU of the multi-GPU path's host logic:

* the slab decomposition's data movement (tests/slab_model.py: send layout,
  all-to-all, y-slab multiplier with global y, reverse transpose, rank-order
  residual) reproduces the single-process oracle's iterate and residuals;
* the NCCL unique id that libusp draws on rank 0 reaches every rank intact
  through torch.distributed (paper_2207_14222_b200.usp broadcast helper).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _model_worker(rank, world, port, shape, n_iter, out_dir):
    import torch.distributed as dist

    _init(rank, world, port)
    from oracle import oracle as O
    from slab_model import delta_form_slab
    from synth import make

    p = make("C3", shape)
    med = np.asarray(p.medium, dtype=np.complex128)
    sp = O.canonical(p.kind, med, 0.95)
    w = O.medium_to_w(p.kind, med)
    nzl = shape[0] // world
    sl = slice(rank * nzl, (rank + 1) * nzl)
    x, hist = delta_form_slab(w[sl], np.asarray(p.source, dtype=np.complex128)[sl], world, rank, shape,
                              p.h, sp.D, sp.sigma, sp.c, p.alpha, n_iter)
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"h{rank}.npy"), hist)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (16, 16, 32)), (4, (16, 32, 16))])
def test_slab_model_matches_oracle(orc, tmp_path, world, shape):
    import torch.multiprocessing as mp
    from synth import make

    n_iter = 12
    mp.spawn(_model_worker, args=(world, _free_port(), shape, n_iter, str(tmp_path)), nprocs=world)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(world)], axis=0)
    hists = [np.load(tmp_path / f"h{r}.npy") for r in range(world)]
    for h in hists[1:]:
        assert np.array_equal(h, hists[0])            # every rank: the same residuals, same stop decision
    p = make("C3", shape)
    med = np.asarray(p.medium, dtype=np.complex128)
    sp = orc.canonical(p.kind, med, 0.95)
    res = orc.fixed_point(orc.medium_to_w(p.kind, med), np.asarray(p.source, dtype=np.complex128), p.h, sp.D,
                          sp.sigma, sp.c, p.alpha, 0.0, n_iter)
    assert np.linalg.norm(x - res.x) <= 1e-11 * np.linalg.norm(res.x)
    assert np.allclose(hists[0][:n_iter], res.hist[:n_iter], rtol=1e-10, atol=1e-14)


def _id_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    _init(rank, world, port)
    from paper_2207_14222_b200.usp import broadcast_unique_id

    idb = broadcast_unique_id()
    with open(os.path.join(out_dir, f"id{rank}.bin"), "wb") as f:
        f.write(bytes(idb))
    dist.barrier()
    dist.destroy_process_group()


def test_unique_id_broadcast(tmp_path):
    import torch.multiprocessing as mp

    from paper_2207_14222_b200 import build as B

    B.build()
    world = 2
    mp.spawn(_id_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world)
    ids = [open(tmp_path / f"id{r}.bin", "rb").read() for r in range(world)]
    assert len(ids[0]) == 128 and any(ids[0]) and ids[1] == ids[0]
