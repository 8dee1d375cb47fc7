"""Thin Python front end of libstencil.so: torch tensors for device memory and streams,
ctypes for the C ABI (include/stencil.h).  Every step of the sweep runs in the CUDA library;
this module only marshals arguments.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from .fd import fd_weights


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _points(pts) -> Tuple[int, Optional[np.ndarray]]:
    if pts is None or len(pts) == 0:
        return 0, None
    a = np.ascontiguousarray(np.asarray(pts, dtype=np.int32).reshape(-1, 3))
    return a.shape[0], a


class Stencil:
    """One plan: grid, stencil and time-tiling configuration on one CUDA device.

    ndim: 2 or 3;  n: GLOBAL interior (nx, ny, nz);  space_order: 2..16 (radius = order/2);
    time_order: 1 heat / 2 damped wave;  t_kernel: on-chip time-tile depth;  t_comm: halo depth
    in steps for z-slabs (rank/nranks).  Layout: see include/stencil.h.
    """

    def __init__(self, ndim: int, n: Sequence[int], space_order: int, time_order: int, dt: float,
                 dx: Sequence[float], t_kernel: int = 1, t_comm: int = 1, rank: int = 0,
                 nranks: int = 1, device: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None,
                 coeffs: Optional[Sequence[float]] = None, no_swap: bool = False,
                 nccl_id: Optional[bytes] = None):
        lib = _lib.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ndim, self.time_order, self.radius = ndim, time_order, space_order // 2
        self.n = tuple(int(v) for v in n)
        c = np.ascontiguousarray(fd_weights(space_order) if coeffs is None else coeffs, dtype=np.float64)
        self._coeffs = c
        cfg = _lib.StConfig()
        cfg.ndim = ndim
        cfg.n[:] = list(self.n)
        cfg.radius = self.radius
        cfg.coeffs = c.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        cfg.time_order = time_order
        cfg.dt = float(dt)
        dxs = list(dx) + [1.0] * (3 - len(dx))
        cfg.dx[:] = [float(v) for v in dxs[:3]]
        cfg.t_kernel, cfg.t_comm = int(t_kernel), int(t_comm)
        cfg.rank, cfg.nranks = int(rank), int(nranks)
        cfg.device = self.device
        cfg.stream = ctypes.c_void_p(self.stream.cuda_stream)
        cfg.flags = _lib.ST_FTZ | (_lib.ST_NO_SWAP if no_swap else 0)
        # library-owned halo exchange (include/stencil.h st_config.nccl_id): NCCL inside the plan
        self._nccl_id = None
        if nccl_id is not None:
            if len(nccl_id) != _lib.ST_NCCL_ID_BYTES:
                raise ValueError("nccl_id must be ST_NCCL_ID_BYTES bytes (stencil_nccl_unique_id)")
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), _lib.ST_NCCL_ID_BYTES)
            cfg.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        self.lib_exchange = nccl_id is not None
        self._cfg = cfg
        h = ctypes.c_void_p()
        _lib.check(lib.stencil_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        padded = (ctypes.c_int64 * 3)()
        origin = (ctypes.c_int64 * 3)()
        zr = (ctypes.c_int64 * 2)()
        _lib.check(lib.stencil_layout(h, padded, origin, zr), h)
        self.X, self.Y, self.Z = padded[0], padded[1], padded[2]
        self.G = origin[2]
        self.z_range = (zr[0], zr[1])
        self.t_kernel, self.t_comm, self.rank, self.nranks = t_kernel, t_comm, rank, nranks

    # ------------------------------------------------------------------ layout helpers
    @property
    def shape(self):
        return (self.Z, self.Y, self.X)

    @property
    def nz_local(self):
        return self.z_range[1] - self.z_range[0]

    def empty(self) -> torch.Tensor:
        return torch.zeros(self.shape, dtype=torch.float32, device=f"cuda:{self.device}")

    def embed(self, interior, ghost_lo: int = 0, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Place an interior array (planes, ny, nx) into the padded layout; its first plane goes
        to array plane G - ghost_lo (so slabs with ghost planes can be embedded directly)."""
        t = torch.as_tensor(interior)
        out = self.empty() if out is None else out
        z0 = self.G - ghost_lo
        out[z0:z0 + t.shape[0], :, :self.n[0]].copy_(t, non_blocking=True)
        return out

    def interior(self, field: torch.Tensor) -> torch.Tensor:
        """View of the owned interior (nz_local, ny, nx)."""
        return field[self.G:self.G + (self.nz_local if self.ndim == 3 else 1), :, :self.n[0]]

    # ------------------------------------------------------------------ run
    def run(self, u_prev: torch.Tensor, u_cur: torch.Tensor, nt: int, vel: Optional[torch.Tensor] = None,
            damp: Optional[torch.Tensor] = None, step0: int = 0, src=None,
            wavelet: Optional[torch.Tensor] = None, rec=None,
            trace: Optional[torch.Tensor] = None, save_every: int = 0,
            snapshots: Optional[torch.Tensor] = None, init=None) -> Optional[torch.Tensor]:
        """Advance (u_prev, u_cur) by nt steps in place (asynchronous on the plan's stream).
        Returns the receiver trace tensor [nt, nrec] (allocated if not given).
        save_every > 0: also store u^{n + j*save_every}, j = 1..nt//save_every, into
        snapshots[j-1] (a [nsnap, Z, Y, X] float32 CUDA tensor; stencil_run_save).
        init = (init_prev, init_cur): start from this kept pair instead of (u_prev, u_cur), which
        then only receive the result (stencil_run_from; heat: init_prev may be None)."""
        init_prev, init_cur = (None, None) if init is None else init
        if init is not None and (init_cur is None or save_every):
            raise ValueError("init needs init_cur and does not combine with snapshots")
        for t in (u_prev, u_cur, vel, damp, wavelet, trace, init_prev, init_cur):
            if t is not None:
                if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
                    raise ValueError("fields/wavelet/trace must be contiguous float32 CUDA tensors")
        for t in (u_prev, u_cur, vel, damp, init_prev, init_cur):
            if t is not None and tuple(t.shape) != self.shape:
                raise ValueError(f"field shape {tuple(t.shape)} != layout {self.shape}")
        nsrc, src_a = _points(src)
        nrec, rec_a = _points(rec)
        if nrec and trace is None:
            trace = torch.zeros((nt, nrec), dtype=torch.float32, device=u_cur.device)
        # the C ABI cannot check buffer lengths: a short trace or wavelet would be overrun
        if nrec and (trace.dim() != 2 or trace.shape[0] < nt or trace.shape[1] != nrec):
            raise ValueError(f"trace must be [>= nt={nt}, nrec={nrec}] (got {tuple(trace.shape)})")
        if nsrc and (wavelet is None or wavelet.dim() != 2 or wavelet.shape[0] < step0 + nt
                     or wavelet.shape[1] != nsrc):
            got = None if wavelet is None else tuple(wavelet.shape)
            raise ValueError(f"wavelet must be [>= step0+nt={step0 + nt}, nsrc={nsrc}] (got {got})")
        lib = _lib.load()
        args = (self._h, _ptr(u_prev), _ptr(u_cur), _ptr(vel), _ptr(damp), int(nt), int(step0), nsrc,
                None if src_a is None else src_a.ctypes.data_as(ctypes.c_void_p), _ptr(wavelet), nrec,
                None if rec_a is None else rec_a.ctypes.data_as(ctypes.c_void_p), _ptr(trace))
        if save_every:
            if snapshots is None or not snapshots.is_cuda or snapshots.dtype != torch.float32 \
                    or not snapshots.is_contiguous() or tuple(snapshots.shape[1:]) != self.shape \
                    or snapshots.shape[0] < nt // save_every:
                raise ValueError("snapshots must be a contiguous float32 CUDA tensor [nt//save_every, Z, Y, X]")
            stride = self.shape[0] * self.shape[1] * self.shape[2]
            st = lib.stencil_run_save(*args, int(save_every), _ptr(snapshots), stride)
        elif init is not None:
            st = lib.stencil_run_from(args[0], _ptr(init_prev), _ptr(init_cur), *args[1:])
        else:
            st = lib.stencil_run(*args)
        _lib.check(st, self._h)
        return trace

    def swapped(self) -> bool:
        """no_swap plans: True if the last run left (u_prev, u_cur) holding (u^{n+nt}, u^{n+nt-1});
        the caller then exchanges its two references (include/stencil.h stencil_swapped)."""
        return _lib.load().stencil_swapped(self._h) == 1

    # ------------------------------------------------------------------ fused halo push
    def peer_counters(self) -> int:
        """Device address of this plan's two inbound push counters (include/stencil.h)."""
        c = ctypes.c_void_p()
        _lib.check(_lib.load().stencil_peer_counters(self._h, ctypes.byref(c)), self._h)
        return int(c.value)

    def set_peer(self, side: int, my_a: torch.Tensor, my_b: torch.Tensor, peer_a: int, peer_b: int,
                 peer_counters: int):
        """Register the neighbour on `side` (0 = rank-1, 1 = rank+1) for the fused halo push:
        my_a/my_b this rank's field pair, peer_* device addresses valid in this process."""
        _lib.check(_lib.load().stencil_set_peer(self._h, int(side), _ptr(my_a), _ptr(my_b),
                                                ctypes.c_void_p(peer_a), ctypes.c_void_p(peer_b),
                                                ctypes.c_void_p(peer_counters)), self._h)

    def ipc_export(self, ptr: int) -> bytes:
        """IPC blob (handle of the allocation holding device address ptr + offset)."""
        blob = ctypes.create_string_buffer(_lib.ST_IPC_BYTES)
        _lib.check(_lib.load().stencil_ipc_export(self._h, ctypes.c_void_p(ptr), blob), self._h)
        return blob.raw

    def ipc_open(self, blob: bytes) -> int:
        """Device address in this process of a peer process's exported pointer."""
        out = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(blob), _lib.ST_IPC_BYTES)
        _lib.check(_lib.load().stencil_ipc_open(self._h, buf, ctypes.byref(out)), self._h)
        return int(out.value)

    def set_timing(self, enable: bool = True):
        _lib.check(_lib.load().stencil_set_timing(self._h, int(enable)), self._h)

    def timing(self):
        """(sweep_ms, sweep_launches, tiled_launches, aux_launches) of the last run (waits for it)."""
        ms = ctypes.c_float()
        n = ctypes.c_int32()
        nt = ctypes.c_int32()
        na = ctypes.c_int32()
        _lib.check(_lib.load().stencil_timing(self._h, ctypes.byref(ms), ctypes.byref(n),
                                              ctypes.byref(nt), ctypes.byref(na)), self._h)
        return float(ms.value), int(n.value), int(nt.value), int(na.value)

    def sync(self):
        _lib.check(_lib.load().stencil_sync(self._h), self._h)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().stencil_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def supported(ndim: int, time_order: int, radius: int, t_kernel: int) -> bool:
    return bool(_lib.load().stencil_supported(ndim, time_order, radius, t_kernel))


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (stencil_nccl_unique_id): rank 0 makes it, every rank passes it as
    Stencil(..., nccl_id=...) to hand the halo exchange to the library."""
    buf = ctypes.create_string_buffer(_lib.ST_NCCL_ID_BYTES)
    _lib.check(_lib.load().stencil_nccl_unique_id(buf))
    return buf.raw
