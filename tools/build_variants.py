"""Build experimental variants of the untiled kernel for a config sweep (see tools/sweep_variants.sh)."""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02347_b200.build import build_variant  # noqa: E402

ONLY = [(3, 1, 6, 1), (3, 1, 4, 1), (3, 1, 8, 1)]
VARIANTS = {
    "base": dict(defines=[], ncw=16),
    "pd6": dict(defines=["-DST_PD=6"], ncw=16),
    "d8": dict(defines=["-DST_T1_DEPTH=8"], ncw=16),
    "d4": dict(defines=["-DST_T1_DEPTH=4"], ncw=16),
    "ncw20": dict(defines=[], ncw=20),
    "ncw24": dict(defines=[], ncw=24),
    "ncw12": dict(defines=[], ncw=12),
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    with cf.ThreadPoolExecutor(2) as ex:
        for n, lib in zip(names, ex.map(lambda n: build_variant(n, only=ONLY, **VARIANTS[n]), names)):
            print(n, lib)
