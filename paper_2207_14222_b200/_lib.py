"""ctypes loader for libusp.so (the in-tree C-ABI library, include/usp.h).

There is no fallback: if the library is missing or fails to load, importing
the package's solver API raises.  Every computation goes through libusp's
CUDA kernels.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libusp.so")

USP_OK = 0
STATUS_NAMES = {0: "USP_OK", 1: "USP_ERR_ARG", 2: "USP_ERR_STATE", 3: "USP_ERR_NOT_CONTRACTIVE",
                4: "USP_ERR_NOT_ACCRETIVE", 5: "USP_ERR_UNSUPPORTED", 6: "USP_ERR_NOMEM",
                7: "USP_ERR_CUDA", 8: "USP_ERR_NCCL", 9: "USP_ERR_NONFINITE"}
TERM_NAMES = {0: "converged", 1: "max_iter", 2: "diverged"}
MEDIUM_K2, MEDIUM_W = 0, 1
C64, R32 = 0, 1
DEVICE, HOST, STAGED = 0, 1, 2


class c128(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class PlanDesc(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("n", ctypes.c_int64 * 3), ("h", ctypes.c_double * 3),
                ("medium", ctypes.c_int), ("dtype", ctypes.c_int), ("D", ctypes.c_double),
                ("sigma", c128), ("c", c128), ("stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p),
                ("virtual_ranks", ctypes.c_int), ("antisymmetric", ctypes.c_int),
                ("tensor_diffusion", ctypes.c_int), ("delta_form", ctypes.c_int), ("r_switch", ctypes.c_double),
                ("dense_source", ctypes.c_int), ("separate_transposes", ctypes.c_int),
                ("complex_path", ctypes.c_int), ("launch_per_pass", ctypes.c_int), ("plane_chain", ctypes.c_int),
                ("test_hooks", ctypes.c_int), ("flat_work", ctypes.c_int)]


HOOK_RANK_FINISH = 1


class USPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


_lib = None

# name -> (restype, argtypes) for every entry point of include/usp.h
SIGNATURES = {
    "usp_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "usp_plan_workspace_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "usp_plan_set_workspace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "usp_local_extent": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "usp_set_potential": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double]),
    "usp_set_tensor_medium": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_double]),
    "usp_get_split": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(c128), ctypes.POINTER(c128),
                                     ctypes.POINTER(c128), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]),
    "usp_set_source": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "usp_iterate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]),
    "usp_residual": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]),
    "usp_residual_history": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_int64)]),
    "usp_get_field": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "usp_staging_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "usp_plan_set_staging": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "usp_stage_inputs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "usp_get_field_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "usp_wait_field": (ctypes.c_int, [ctypes.c_void_p]),
    "usp_profile_enable": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "usp_profile_read": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int)]),
    "usp_launch_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "usp_iteration_form": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]),
    "usp_work_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "usp_transport": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "usp_shared_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "usp_shared_free": (ctypes.c_int, [ctypes.c_void_p]),
    "usp_plan_destroy": (None, [ctypes.c_void_p]),
    "usp_comm_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte)]),
    "usp_comm_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte), ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_void_p)]),
    "usp_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "usp_krylov_workspace_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "usp_krylov_set_workspace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "usp_bicgstab": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]),
    "usp_gmres_workspace_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "usp_gmres_set_workspace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]),
    "usp_gmres": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]),
    "usp_last_error": (ctypes.c_char_p, []),
    "usp_version": (ctypes.c_char_p, []),
}


def _nccl_path_hint():
    """Point libusp's run-time NCCL loader at the torch wheel's libnccl.so.2
    (used only by multi-GPU plans)."""
    if "USP_NCCL_LIB" in os.environ:
        return
    try:
        import nvidia.nccl as nn

        for d in nn.__path__:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["USP_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def load():
    """Load libusp.so (building it first if it is absent).  Raises on failure."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from .build import build

        build()
    _nccl_path_hint()
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != USP_OK:
        msg = load().usp_last_error().decode(errors="replace")
        raise USPError(status, msg)
