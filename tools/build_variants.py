"""Build experimental variants of the sweep kernels for a config sweep (see tools/gpu_variants.sh).

    python tools/build_variants.py NAME [NAME ...]
"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02347_b200.build import build_variant  # noqa: E402

ONLY = [(3, 1, 6, 1), (3, 1, 4, 1), (3, 1, 8, 1), (3, 1, 4, 2), (3, 0, 1, 1), (3, 0, 1, 2), (3, 0, 1, 4),
        (3, 1, 1, 1), (3, 1, 1, 2), (3, 1, 2, 1), (3, 1, 2, 2)]
VARIANTS = {
    "base": dict(defines=[]),
    "rot": dict(defines=["-DST_ROT1=1", "-DST_ROT2=1"]),
    "rot1": dict(defines=["-DST_ROT1=1"]),
    "rot2": dict(defines=["-DST_ROT2=1"]),
    "unr": dict(defines=["-DST_ROT2=0"]),
    "de4": dict(defines=["-DST_DE2=4", "-DST_DL2=2"]),
    "unr_de4": dict(defines=["-DST_ROT2=0", "-DST_DE2=4", "-DST_DL2=2"]),
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    with cf.ThreadPoolExecutor(2) as ex:
        for n, lib in zip(names, ex.map(lambda n: build_variant(n, only=ONLY, **VARIANTS[n]), names)):
            print(n, lib)
