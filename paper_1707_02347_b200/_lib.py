"""ctypes binding of libstencil.so (include/stencil.h).  Argument marshalling only.

The library is the product: there is no CPU fallback.  If libstencil.so is missing or cannot
be loaded, every entry point raises -- loudly -- instead of computing anything elsewhere.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ST_LIB") or os.path.join(HERE, "libstencil.so")   # ST_LIB: experiment builds

ST_OK, ST_EINVAL, ST_ENOMEM, ST_ECUDA, ST_ENCCL, ST_EUNSUPPORTED, ST_ESTATE = 0, 1, 2, 3, 4, 5, 6
ST_FTZ = 1
ST_NO_SWAP = 2
STATUS_NAMES = {0: "ST_OK", 1: "ST_EINVAL", 2: "ST_ENOMEM", 3: "ST_ECUDA", 4: "ST_ENCCL",
                5: "ST_EUNSUPPORTED", 6: "ST_ESTATE"}

# Every symbol include/stencil.h declares (checked by tests/test_abi_symbols.py).
EXPORTS = ("stencil_create", "stencil_layout", "stencil_run", "stencil_run_save", "stencil_run_from",
           "stencil_sync",
           "stencil_destroy", "stencil_last_error", "stencil_supported", "stencil_abi_version",
           "stencil_set_timing", "stencil_timing", "stencil_swapped", "stencil_peer_counters",
           "stencil_set_peer", "stencil_ipc_export", "stencil_ipc_open", "stencil_nccl_unique_id")
ST_IPC_BYTES = 72
ST_NCCL_ID_BYTES = 128


class StConfig(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("n", ctypes.c_int64 * 3),
        ("radius", ctypes.c_int32),
        ("coeffs", ctypes.POINTER(ctypes.c_double)),
        ("time_order", ctypes.c_int32),
        ("dt", ctypes.c_double),
        ("dx", ctypes.c_double * 3),
        ("t_kernel", ctypes.c_int32),
        ("t_comm", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("nccl_id", ctypes.c_void_p),
    ]


class StencilError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    """Load libstencil.so (raises if it is absent: build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not found: the CUDA extension is not built "
                           "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                           "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.stencil_create.argtypes = [ctypes.POINTER(StConfig), ctypes.POINTER(P)]
    lib.stencil_create.restype = ctypes.c_int
    lib.stencil_layout.argtypes = [P, ctypes.c_int64 * 3, ctypes.c_int64 * 3, ctypes.c_int64 * 2]
    lib.stencil_layout.restype = ctypes.c_int
    lib.stencil_run.argtypes = [P, P, P, P, P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, P, P,
                                ctypes.c_int32, P, P]
    lib.stencil_run.restype = ctypes.c_int
    lib.stencil_run_save.argtypes = lib.stencil_run.argtypes + [ctypes.c_int32, P, ctypes.c_int64]
    lib.stencil_run_save.restype = ctypes.c_int
    lib.stencil_run_from.argtypes = lib.stencil_run.argtypes[:1] + [P, P] + lib.stencil_run.argtypes[1:]
    lib.stencil_run_from.restype = ctypes.c_int
    lib.stencil_sync.argtypes = [P]
    lib.stencil_sync.restype = ctypes.c_int
    lib.stencil_destroy.argtypes = [P]
    lib.stencil_destroy.restype = None
    lib.stencil_last_error.argtypes = [P]
    lib.stencil_last_error.restype = ctypes.c_char_p
    lib.stencil_supported.argtypes = [ctypes.c_int32] * 4
    lib.stencil_supported.restype = ctypes.c_int32
    lib.stencil_set_timing.argtypes = [P, ctypes.c_int32]
    lib.stencil_set_timing.restype = ctypes.c_int
    lib.stencil_timing.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    lib.stencil_timing.restype = ctypes.c_int
    lib.stencil_peer_counters.argtypes = [P, ctypes.POINTER(P)]
    lib.stencil_peer_counters.restype = ctypes.c_int
    lib.stencil_set_peer.argtypes = [P, ctypes.c_int32, P, P, P, P, P]
    lib.stencil_set_peer.restype = ctypes.c_int
    lib.stencil_ipc_export.argtypes = [P, P, P]
    lib.stencil_ipc_export.restype = ctypes.c_int
    lib.stencil_ipc_open.argtypes = [P, P, ctypes.POINTER(P)]
    lib.stencil_ipc_open.restype = ctypes.c_int
    lib.stencil_swapped.argtypes = [P]
    lib.stencil_swapped.restype = ctypes.c_int32
    lib.stencil_abi_version.argtypes = []
    lib.stencil_abi_version.restype = ctypes.c_int32
    lib.stencil_nccl_unique_id.argtypes = [P]
    lib.stencil_nccl_unique_id.restype = ctypes.c_int
    _lib = lib
    return lib


def check(status: int, plan=None):
    if status != ST_OK:
        msg = load().stencil_last_error(plan)
        raise StencilError(status, (msg or b"").decode(errors="replace"))
