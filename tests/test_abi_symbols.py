"""CPU checks of the boundary: libstencil.so loads, exports every symbol include/stencil.h
declares, answers its pure host queries, and fails cleanly (no crash) without a GPU.
Also: the product's FD weights (Fornberg, exact) equal the oracle's closed form."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

import oracle
from paper_1707_02347_b200 import _lib
from paper_1707_02347_b200.fd import fornberg_weights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stencil.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(stencil_[a-z_]+)\s*\(", txt)))


def test_header_declares_binding_exports():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_host_queries():
    lib = _lib.load()
    assert lib.stencil_abi_version() == 105
    for r in range(1, 9):
        for to in (1, 2):
            assert lib.stencil_supported(3, to, r, 1) == 1
            assert lib.stencil_supported(3, to, r, 2) == 1
            assert lib.stencil_supported(2, to, r, 1) == 1
    assert lib.stencil_supported(3, 1, 1, 4) == 1
    assert lib.stencil_supported(3, 2, 9, 1) == 0
    assert lib.stencil_supported(4, 2, 1, 1) == 0


def _cfg(**kw):
    c = _lib.StConfig()
    coeffs = np.array([-2.0, 1.0])
    c.ndim = kw.get("ndim", 3)
    c.n[:] = kw.get("n", [16, 16, 16])
    c.radius = kw.get("radius", 1)
    c.coeffs = coeffs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if kw.get("coeffs", True) else None
    c.time_order = kw.get("time_order", 1)
    c.dt = 0.1
    c.dx[:] = [1.0, 1.0, 1.0]
    c.t_kernel = kw.get("t_kernel", 1)
    c.t_comm = kw.get("t_comm", 1)
    c.rank, c.nranks = kw.get("rank", 0), kw.get("nranks", 1)
    c.device = 0
    c.stream = None
    c.flags = kw.get("flags", _lib.ST_FTZ)
    return c, coeffs


@pytest.mark.parametrize("kw,status", [
    (dict(radius=0), _lib.ST_EINVAL),
    (dict(radius=9), _lib.ST_EINVAL),
    (dict(ndim=4), _lib.ST_EINVAL),
    (dict(coeffs=False), _lib.ST_EINVAL),
    (dict(t_kernel=0), _lib.ST_EINVAL),
    (dict(nranks=2, n=[16, 16, 15]), _lib.ST_EINVAL),
    (dict(nranks=2, rank=2), _lib.ST_EINVAL),
    (dict(nranks=2, t_kernel=2, t_comm=3), _lib.ST_EINVAL),
    (dict(nranks=4, t_comm=5), _lib.ST_EINVAL),              # ghost depth 5 > slab of 4 planes
    (dict(flags=0), _lib.ST_EUNSUPPORTED),
    (dict(radius=3, t_kernel=8), _lib.ST_EUNSUPPORTED),
])
def test_create_rejects_bad_config(kw, status):
    lib = _lib.load()
    c, keep = _cfg(**kw)
    h = ctypes.c_void_p(123)
    st = lib.stencil_create(ctypes.byref(c), ctypes.byref(h))
    assert st == status
    assert h.value is None
    assert len(lib.stencil_last_error(None)) > 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_create_without_gpu_fails_cleanly():
    lib = _lib.load()
    c, keep = _cfg()
    h = ctypes.c_void_p()
    st = lib.stencil_create(ctypes.byref(c), ctypes.byref(h))
    assert st == _lib.ST_ECUDA
    assert b"cuda" in lib.stencil_last_error(None).lower()


def test_null_arguments():
    lib = _lib.load()
    assert lib.stencil_create(None, None) == _lib.ST_EINVAL
    assert lib.stencil_run(None, None, None, None, None, 1, 0, 0, None, None, 0, None, None) == _lib.ST_EINVAL
    assert lib.stencil_sync(None) == _lib.ST_EINVAL
    lib.stencil_destroy(None)


@pytest.mark.parametrize("order", range(2, 17, 2))
def test_product_fd_weights_equal_oracle(order):
    assert tuple(fornberg_weights(order)) == tuple(oracle.fd_weights_exact(order))


def test_nccl_unique_id_host_only():
    """stencil_nccl_unique_id (library-owned exchange) needs no GPU: the NCCL the process loads
    (torch's libnccl.so.2) makes the id rank 0 broadcasts."""
    import torch  # noqa: F401  (loads libnccl.so.2 into the process)
    lib = _lib.load()
    buf = ctypes.create_string_buffer(_lib.ST_NCCL_ID_BYTES)
    st = lib.stencil_nccl_unique_id(buf)
    if st == _lib.ST_ENCCL:
        pytest.skip(lib.stencil_last_error(None).decode())
    assert st == _lib.ST_OK and any(buf.raw)
    assert lib.stencil_nccl_unique_id(None) == _lib.ST_EINVAL
