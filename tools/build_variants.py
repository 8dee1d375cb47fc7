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
    "de3dl5": dict(defines=["-DST_DE2=3", "-DST_DL2=5"]),
    "de3dl4": dict(defines=["-DST_DE2=3", "-DST_DL2=4"]),
    "de4dl3": dict(defines=["-DST_DE2=4", "-DST_DL2=3"]),
    "de3dl5rot": dict(defines=["-DST_DE2=3", "-DST_DL2=5", "-DST_ROT2=1"]),
    "w1": dict(defines=["-DST_WAIT2=1"]),
    "w2": dict(defines=["-DST_WAIT2=2"]),
    "w1dl3": dict(defines=["-DST_WAIT2=1", "-DST_DL2=3"]),
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    with cf.ThreadPoolExecutor(2) as ex:
        for n, lib in zip(names, ex.map(lambda n: build_variant(n, only=ONLY, **VARIANTS[n]), names)):
            print(n, lib)
