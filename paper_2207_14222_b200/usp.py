"""Thin Python binding of libusp (include/usp.h): argument marshalling only.

PyTorch supplies device memory (the workspace and field tensors) and the
stream; every step of the method runs in libusp's sm_100a kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

_TERM = L.TERM_NAMES


@dataclass
class Split:
    sigma: complex
    c: complex
    centre: complex
    radius: float
    max_abs_V: float


def _numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") and callable(a.numel) else int(np.asarray(a).size)


def _ptr_where(a, want_dtype):
    """(pointer, where, keepalive) for a torch tensor or numpy array."""
    try:
        import torch
    except Exception:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        tdt = {"c64": torch.complex64, "r32": torch.float32}[want_dtype]
        if a.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr()), (L.DEVICE if a.is_cuda else L.HOST), a
    arr = np.asarray(a)
    ndt = {"c64": np.complex64, "r32": np.float32}[want_dtype]
    if arr.dtype != ndt or not arr.flags.c_contiguous:
        raise TypeError(f"expected a C-contiguous {np.dtype(ndt)} array, got {arr.dtype}")
    return ctypes.c_void_p(arr.ctypes.data), L.HOST, arr


class Plan:
    """One solver plan for a grid of ``shape`` (C order, x last).

    kind='helmholtz': medium is k^2(r) (Eq. 8); kind='diffusion':
    medium is mu_a(r) (§3.2, scalar D).  dtype 'c64' (complex64 arrays) or
    'r32' (float32 arrays, diffusion with real data).

    Slab decomposition (3-D): ``comm`` = a communicator from
    :func:`comm_init` splits the grid into z-slabs over its ranks (one GPU
    per rank; arrays are the rank's slab, ``local_shape``);
    ``virtual_ranks=P`` runs the same decomposition with P slabs on one GPU
    (transposes as device copies; arrays are the full grid).

    ``antisymmetric=True`` solves the antisymmetrised system of Eq. 9-10
    (accretive for any problem, e.g. gain media); ``get_field`` returns x.

    Options (usp_plan_desc; the defaults are the library's):
    ``delta_form`` (Delta-form recurrence from the first iteration instead of
    the x-form while r >= ``r_switch``, R-30), ``dense_source`` (no
    sparse-source x pass, R-31), ``separate_transposes`` (NCCL all-to-all
    transposes of the slab decomposition instead of the fused peer stores),
    ``complex_path`` (float32 diffusion data on the complex path),
    ``launch_per_pass`` (2-D: one launch per pass instead of the persistent
    solver), ``plane_chain`` (the plane-chained pass on 1024^2-plane
    grids instead of one sweep per FFT pass), ``flat_work`` (the z pass in place
    on the [z][y][x] chain buffer instead of the z-pair buffer),
    ``test_hooks`` (USP_HOOK_* bits; tests only).
    """

    def __init__(self, shape: Sequence[int], kind: str = "helmholtz", h: Optional[Sequence[float]] = None,
                 D: float = 1.0, sigma: complex = 0j, c: complex = 1 + 0j, dtype: str = "c64",
                 stream=None, device=None, comm=None, virtual_ranks: int = 0, antisymmetric: bool = False,
                 tensor_diffusion: bool = False, delta_form: bool = False, r_switch: float = 0.0,
                 dense_source: bool = False, separate_transposes: bool = False, complex_path: bool = False,
                 launch_per_pass: bool = False, plane_chain: bool = False, test_hooks: int = 0,
                 flat_work: bool = False):
        import torch

        self.lib = L.load()
        self.shape = tuple(int(s) for s in shape)
        self.ndim = len(self.shape)
        self.kind = kind
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        d = L.PlanDesc()
        d.ndim = self.ndim
        rev = list(reversed(self.shape)) + [1] * (3 - self.ndim)
        hh = list(reversed(h)) if h is not None else [1.0] * self.ndim
        hh += [1.0] * (3 - self.ndim)
        for a in range(3):
            d.n[a] = rev[a]
            d.h[a] = float(hh[a])
        d.medium = L.MEDIUM_K2 if kind == "helmholtz" else L.MEDIUM_W
        d.dtype = L.C64 if dtype == "c64" else L.R32
        d.D = float(D)
        d.sigma = L.c128(float(np.real(sigma)), float(np.imag(sigma)))
        d.c = L.c128(float(np.real(c)), float(np.imag(c)))
        d.stream = ctypes.c_void_p(self.stream.cuda_stream)
        d.nccl_comm = comm.handle if comm is not None else None
        d.virtual_ranks = int(virtual_ranks)
        d.antisymmetric = int(bool(antisymmetric))
        d.tensor_diffusion = int(bool(tensor_diffusion))
        d.delta_form = int(bool(delta_form))
        d.r_switch = float(r_switch)
        d.dense_source = int(bool(dense_source))
        d.separate_transposes = int(bool(separate_transposes))
        d.complex_path = int(bool(complex_path))
        d.launch_per_pass = int(bool(launch_per_pass))
        d.plane_chain = int(bool(plane_chain))
        d.test_hooks = int(test_hooks)
        d.flat_work = int(bool(flat_work))
        if tensor_diffusion:
            d.dtype = L.R32
            self.dtype = "r32"
        self.comm = comm
        self.desc = d
        h_ = ctypes.c_void_p()
        L.check(self.lib.usp_plan_create(ctypes.byref(d), ctypes.byref(h_)))
        self.handle = h_
        nbytes = ctypes.c_size_t()
        L.check(self.lib.usp_plan_workspace_size(self.handle, ctypes.byref(nbytes)))
        self._ws_raw = None
        if comm is not None:
            # slab decomposition over ranks: a workspace of its own (usp_shared_alloc:
            # ncclMemAlloc, so NCCL can register it as a window for the fused
            # transposes, else cudaMalloc, which CUDA IPC can map whatever torch's
            # allocator settings)
            with torch.cuda.device(self.device):
                ptr = ctypes.c_void_p()
                L.check(self.lib.usp_shared_alloc(int(nbytes.value), ctypes.byref(ptr)))
                self._ws_raw = ptr
            self.workspace = None
            ws_ptr = self._ws_raw
        else:
            self.workspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
            ws_ptr = ctypes.c_void_p(self.workspace.data_ptr())
        L.check(self.lib.usp_plan_set_workspace(self.handle, ws_ptr, int(nbytes.value)))
        z0, nzl = ctypes.c_int64(), ctypes.c_int64()
        L.check(self.lib.usp_local_extent(self.handle, ctypes.byref(z0), ctypes.byref(nzl)))
        self.z0 = int(z0.value)
        self.local_shape = ((int(nzl.value),) + self.shape[1:]) if self.ndim == 3 else self.shape
        self.staging = None
        self._staged_keep = []   # host inputs of pending stage_inputs copies (until set_source("staged"))
        self._out_keep = []      # host outputs of pending get_field_async copies (until wait_field)

    # -- setup ---------------------------------------------------------------
    def stage_inputs(self, medium, source):
        """usp_stage_inputs: start copying the NEXT problem's medium and source
        (host arrays, ideally pinned) into the staging area on the plan's copy
        stream; returns at once.  Then call set_potential("staged") and
        set_source("staged").  The host buffers must stay untouched until
        set_source("staged") has returned."""
        self._ensure_staging()
        pm, wm, km = _ptr_where(medium, self.dtype)
        ps, ws, ks = _ptr_where(source, self.dtype)
        if wm != L.HOST or ws != L.HOST:
            raise ValueError("stage_inputs takes host buffers")
        n = int(np.prod(self.local_shape))
        if _numel(km) != n or _numel(ks) != n:
            raise ValueError(f"stage_inputs needs {n} elements per array")
        L.check(self.lib.usp_stage_inputs(self.handle, pm, ps))
        self._staged_keep.append((km, ks))   # the copies read them asynchronously

    def _ensure_staging(self):
        if self.staging is None:
            import torch

            nbytes = ctypes.c_size_t()
            L.check(self.lib.usp_staging_size(self.handle, 1, ctypes.byref(nbytes)))   # with the read-back slot
            self.staging = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
            L.check(self.lib.usp_plan_set_staging(self.handle, ctypes.c_void_p(self.staging.data_ptr()),
                                                  int(nbytes.value)))

    def get_field_async(self, out):
        """usp_get_field_async: start copying x_k into the host array `out`
        (pinned for full speed) on the plan's read-back stream; call
        wait_field() before reading `out`."""
        self._ensure_staging()
        ptr, where, keep = _ptr_where(out, self.dtype)
        if where != L.HOST:
            raise ValueError("get_field_async writes host memory")
        n = int(np.prod(self.local_shape))
        if _numel(keep) != n:
            raise ValueError(f"get_field_async needs a host array of {n} elements, got {_numel(keep)}")
        L.check(self.lib.usp_get_field_async(self.handle, ptr))
        self._out_keep.append(keep)   # alive until wait_field()

    def wait_field(self):
        L.check(self.lib.usp_wait_field(self.handle))
        self._out_keep.clear()

    def set_potential(self, medium, target_norm: float = 0.95):
        if isinstance(medium, str) and medium == "staged":
            L.check(self.lib.usp_set_potential(self.handle, None, L.STAGED, float(target_norm)))
            return self.split
        ptr, where, keep = _ptr_where(medium, self.dtype)
        L.check(self.lib.usp_set_potential(self.handle, ptr, where, float(target_norm)))
        del keep
        return self.split

    def set_tensor_medium(self, mu, D, target_norm: float = 0.95):
        """Tensor-diffusion plans (§3.2): mu_a [shape] and D [shape + (d, d)]
        (symmetric positive definite), packed for usp_set_tensor_medium."""
        import torch

        d = self.ndim
        idx = [(0, 0), (0, 1), (1, 1)] if d == 2 else [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
        if isinstance(D, torch.Tensor):
            pk = torch.stack([D[..., i, j] for i, j in idx], dim=-1).to(torch.float32).contiguous()
        else:
            pk = np.ascontiguousarray(np.stack([np.asarray(D)[..., i, j] for i, j in idx], axis=-1), dtype=np.float32)
        mptr, where, k1 = _ptr_where(mu, "r32")
        dptr, where2, k2 = _ptr_where(pk, "r32")
        if where != where2:
            raise ValueError("mu and D must both be host or both device arrays")
        L.check(self.lib.usp_set_tensor_medium(self.handle, mptr, dptr, where, float(target_norm)))
        del k1, k2
        return self.split

    @property
    def split(self) -> Split:
        s, c, ce = L.c128(), L.c128(), L.c128()
        r, v = ctypes.c_double(), ctypes.c_double()
        L.check(self.lib.usp_get_split(self.handle, ctypes.byref(s), ctypes.byref(c), ctypes.byref(ce),
                                       ctypes.byref(r), ctypes.byref(v)))
        return Split(complex(s.re, s.im), complex(c.re, c.im), complex(ce.re, ce.im), r.value, v.value)

    def set_source(self, src):
        if isinstance(src, str) and src == "staged":
            L.check(self.lib.usp_set_source(self.handle, None, L.STAGED))
            # usp_set_source returns after its setup ran on the plan stream: the
            # oldest staged pair has been copied from the host
            if self._staged_keep:
                self._staged_keep.pop(0)
            return
        ptr, where, keep = _ptr_where(src, self.dtype)
        L.check(self.lib.usp_set_source(self.handle, ptr, where))
        del keep

    # -- iteration -----------------------------------------------------------
    def iterate(self, n_max: int, alpha: float = 0.75, tol: float = 0.0) -> Tuple[int, str]:
        nd = ctypes.c_int64()
        term = ctypes.c_int()
        L.check(self.lib.usp_iterate(self.handle, int(n_max), float(alpha), float(tol), ctypes.byref(nd),
                                     ctypes.byref(term)))
        return int(nd.value), _TERM[term.value]

    def bicgstab(self, n_max: int, tol: float = 0.0) -> Tuple[int, str]:
        """BiCGSTAB on the preconditioned system (usp_bicgstab); starts from
        x_0 = 0 right after set_source.  Allocates the Krylov workspace (5
        complex64 fields) on first use.  Returns (passes, termination)."""
        import torch

        if getattr(self, "kworkspace", None) is None:
            nbytes = ctypes.c_size_t()
            L.check(self.lib.usp_krylov_workspace_size(self.handle, ctypes.byref(nbytes)))
            self.kworkspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
            L.check(self.lib.usp_krylov_set_workspace(self.handle, ctypes.c_void_p(self.kworkspace.data_ptr()),
                                                      int(nbytes.value)))
        nd = ctypes.c_int64()
        term = ctypes.c_int()
        L.check(self.lib.usp_bicgstab(self.handle, int(n_max), float(tol), ctypes.byref(nd), ctypes.byref(term)))
        return int(nd.value), _TERM[term.value]

    def gmres(self, m: int, n_max: int, tol: float = 0.0) -> Tuple[int, str]:
        """Restarted GMRES(m) on the preconditioned system (usp_gmres); starts
        from x_0 = 0 right after set_source.  Allocates the GMRES workspace
        (m + 2 complex64 fields) for this m on first use.  Returns (Arnoldi
        steps, termination)."""
        import torch

        if getattr(self, "gworkspace_m", None) != m:
            nbytes = ctypes.c_size_t()
            L.check(self.lib.usp_gmres_workspace_size(self.handle, int(m), ctypes.byref(nbytes)))
            self.gworkspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
            L.check(self.lib.usp_gmres_set_workspace(self.handle, int(m), ctypes.c_void_p(self.gworkspace.data_ptr()),
                                                     int(nbytes.value)))
            self.gworkspace_m = m
        nd = ctypes.c_int64()
        term = ctypes.c_int()
        L.check(self.lib.usp_gmres(self.handle, int(n_max), float(tol), ctypes.byref(nd), ctypes.byref(term)))
        return int(nd.value), _TERM[term.value]

    def residual(self) -> Tuple[float, float, int]:
        r, a, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        L.check(self.lib.usp_residual(self.handle, ctypes.byref(r), ctypes.byref(a), ctypes.byref(k)))
        return r.value, a.value, int(k.value)

    def history(self) -> np.ndarray:
        n = ctypes.c_int64()
        L.check(self.lib.usp_residual_history(self.handle, None, 0, ctypes.byref(n)))
        buf = np.zeros(int(n.value), dtype=np.float64)
        L.check(self.lib.usp_residual_history(self.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              buf.size, ctypes.byref(n)))
        return buf

    def get_field(self, out=None):
        import torch

        if out is None:
            tdt = torch.complex64 if self.dtype == "c64" else torch.float32
            out = torch.empty(self.local_shape, dtype=tdt, device=self.device)
        ptr, where, keep = _ptr_where(out, self.dtype)
        L.check(self.lib.usp_get_field(self.handle, ptr, where))
        return out

    # -- instrumentation -----------------------------------------------------
    def profile(self, enable: bool = True):
        L.check(self.lib.usp_profile_enable(self.handle, int(enable)))

    def profile_read(self):
        cap = 16
        names = (ctypes.c_char * 32 * cap)()
        ms = (ctypes.c_double * cap)()
        cnt = (ctypes.c_int64 * cap)()
        n = ctypes.c_int()
        L.check(self.lib.usp_profile_read(self.handle, cap, names, ms, cnt, ctypes.byref(n)))
        return {bytes(names[i]).split(b"\0", 1)[0].decode(): (ms[i], int(cnt[i])) for i in range(n.value)}

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        L.check(self.lib.usp_launch_count(self.handle, ctypes.byref(n)))
        return int(n.value)

    def iteration_form(self):
        """(x-form plan?, currently in the x-form?, r_switch) -- usp_iteration_form."""
        xf, fm, rs, sl = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        L.check(self.lib.usp_iteration_form(self.handle, ctypes.byref(xf), ctypes.byref(fm), ctypes.byref(rs),
                                            ctypes.byref(sl)))
        return bool(xf.value), bool(fm.value), float(rs.value)

    def work_layout(self) -> str:
        """"z-pair" or "flat": the chain buffer the z pass runs on (usp_work_layout)."""
        zp = ctypes.c_int()
        L.check(self.lib.usp_work_layout(self.handle, ctypes.byref(zp)))
        return "z-pair" if zp.value else "flat"

    TRANSPORTS = ("none", "virtual", "virtual-copy", "nccl-window", "cuda-ipc", "nccl-alltoall")

    def transport(self) -> str:
        """How the slab transposes move data (usp_transport): "none" (one slab),
        "virtual" / "virtual-copy" (virtual slabs, fused / device copies),
        "nccl-window", "cuda-ipc" (fused peer stores) or "nccl-alltoall"."""
        k = ctypes.c_int()
        L.check(self.lib.usp_transport(self.handle, ctypes.byref(k)))
        return self.TRANSPORTS[k.value]

    def source_lines(self) -> int:
        """Number of x-lines carrying the source when the x-form skips the
        dense s field (reading R-31), else 0."""
        xf, fm, rs, sl = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        L.check(self.lib.usp_iteration_form(self.handle, ctypes.byref(xf), ctypes.byref(fm), ctypes.byref(rs),
                                            ctypes.byref(sl)))
        return int(sl.value)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.usp_plan_destroy(self.handle)
            self.handle = None
        if getattr(self, "_ws_raw", None) is not None:
            L.check(self.lib.usp_shared_free(self._ws_raw))
            self._ws_raw = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """NCCL communicator of libusp's slab decomposition (usp_comm_init).
    The 128-byte unique id travels over torch.distributed (any backend)."""

    def __init__(self, handle, nranks: int, rank: int):
        self.handle = handle
        self.nranks = nranks
        self.rank = rank

    def close(self):
        if getattr(self, "handle", None):
            L.check(L.load().usp_comm_destroy(self.handle))
            self.handle = None


def broadcast_unique_id(group=None):
    """Rank 0 of the torch.distributed ``group`` draws an NCCL unique id
    (usp_comm_unique_id); every rank returns the same 128 bytes."""
    import torch
    import torch.distributed as dist

    lib = L.load()
    idbuf = (ctypes.c_ubyte * 128)()
    if dist.get_rank(group) == 0:
        L.check(lib.usp_comm_unique_id(idbuf))
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0, group=group)
    return (ctypes.c_ubyte * 128)(*t.cpu().tolist())


def comm_init(group=None) -> Comm:
    """Collective over the torch.distributed ``group``: every rank joins the
    NCCL communicator of libusp's slab decomposition on its current CUDA
    device."""
    import torch.distributed as dist

    idbuf = broadcast_unique_id(group)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    h = ctypes.c_void_p()
    L.check(L.load().usp_comm_init(idbuf, world, rank, ctypes.byref(h)))
    return Comm(h, world, rank)


def solve(medium, source, kind: str = "helmholtz", alpha: float = 0.75, tol: float = 0.0, n_iter: int = 100,
          target_norm: float = 0.95, h=None, D: float = 1.0, dtype: str = "c64", sigma=None, c=None):
    """Convenience: plan + canonical form + source + Algorithm 1.  Returns
    (x, n_done, term, plan)."""
    shape = tuple(np.shape(medium)) if not hasattr(medium, "shape") else tuple(medium.shape)
    plan = Plan(shape, kind=kind, h=h, D=D, dtype=dtype,
                sigma=0j if sigma is None else sigma, c=1 + 0j if c is None else c)
    plan.set_potential(medium, target_norm if sigma is None else -1.0)
    plan.set_source(source)
    n, term = plan.iterate(n_iter, alpha, tol)
    return plan.get_field(), n, term, plan
