"""B200-native time-tiled finite-difference stencil sweep (arXiv 1707.02347 hot path).

    from paper_1707_02347_b200 import Stencil
    st = Stencil(3, (512, 512, 512), space_order=8, time_order=2, dt=dt, dx=(10, 10, 10), t_kernel=2)
    st.run(u_prev, u_cur, nt=500, vel=vel, damp=damp, src=[(256, 256, 256)], wavelet=w)

The compute path is libstencil.so (CUDA, sm_100a); see include/stencil.h and DESIGN.md.
Importing this package does not load the library; the first Stencil(...) does, and fails
loudly if it is not built.
"""
from .fd import fd_weights, fornberg_weights  # noqa: F401


def __getattr__(name):
    if name in ("Stencil", "supported"):
        from . import stencil as _s
        return getattr(_s, name)
    raise AttributeError(name)


__all__ = ["Stencil", "supported", "fd_weights", "fornberg_weights"]
