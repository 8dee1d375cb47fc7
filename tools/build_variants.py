"""Build experimental variants of the sweep kernels for a config sweep (see tools/gpu_variants.sh).

    python tools/build_variants.py NAME [NAME ...]
"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02347_b200.build import build_variant  # noqa: E402

ONLY = [(3, 1, R, TK) for R in range(1, 9) for TK in (1, 2)] + [(3, 0, 1, 1), (3, 0, 1, 2), (3, 0, 1, 4)]
VARIANTS = {
    "base": dict(defines=[]),
    "w12v2p3": dict(defines=["-DST_PD=3"], t1=(12, 2)),
    "w12v2p4": dict(defines=["-DST_PD=4"], t1=(12, 2)),
    "w12v2p2": dict(defines=["-DST_PD=2"], t1=(12, 2)),
    "w12v2p3d4": dict(defines=["-DST_PD=3", "-DST_T1_DEPTH=4"], t1=(12, 2)),
    "w10v2p3": dict(defines=["-DST_PD=3"], t1=(10, 2)),
    "w14v2p2": dict(defines=["-DST_PD=2"], t1=(14, 2)),
    "w8v2p4": dict(defines=["-DST_PD=4"], t1=(8, 2)),
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    with cf.ThreadPoolExecutor(2) as ex:
        for n, lib in zip(names, ex.map(lambda n: build_variant(n, only=ONLY, **VARIANTS[n]), names)):
            print(n, lib)
