"""Build libstencil.so (sm_100a) in-tree: generated kernel-instance TUs + abi.cu, nvcc in parallel.

python -m paper_1707_02347_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libstencil.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(HERE, "..", "include")]


def _vy_nwy(ndim: int, R: int, TK: int):
    """Register blocking of the first time-tiled kernel (sweep.cuh): queues hold TK*(2R+1)*VY
    packed pairs per thread."""
    if ndim == 2:
        return 4, 8
    if TK * (2 * R + 1) * 4 <= 72:
        return 4, 8
    return 2, 12


NCW_T1 = 16   # consumer warps (= tile rows) of the untiled warp-specialised kernel (2-D, R = 8)


def _t1_geom(ndim: int, wave: int, R: int):
    """(consumer warps, rows per warp) of the untiled kernel.  Two rows per warp share their
    y-neighbour loads and give two independent FMA chains, which pays for the 3-D wave at
    R = 3..7 (C5 SO12: 247 -> 260-280 GPts/s); at R = 8 the doubled z-queue no longer fits the
    128-register budget of 13 warps, and the heat / low-order sweeps are already at the HBM
    roof with one row per warp (heat C2: 596 vs 511 GPts/s).  Measured, DESIGN.md §10."""
    if ndim == 3 and wave and 3 <= R <= 7:
        return 12, 2
    return NCW_T1, 1

# kernel kinds: 1 = sweep1 (untiled, warp-specialised), 3 = sweep1s (untiled, static 2r+1 ring),
#               2 = sweep2 (time-tiled, warp-specialised, overlapped tiles),
#               4 = sweepx (time-tiled T_k = 2 as L1/L2 untiled sweeps chained through L2),
#               0 = sweep (first time-tiled kernel; 2-D and the shapes sweep2 does not fit)
def _sweep2_oy(wave: int, R: int, TK: int):
    """Output rows of the sweep2 (one warp group per level) instance, or None if it does not fit
    (<= 31 consumer warps of two rows; wave only two levels)."""
    if TK == 2 and R <= 4:
        # measured (DESIGN.md §10, 512^3 x 200 steps, GPts/s): wave SO2 OY 16/14/12/10/8 ->
        # 381/416/423/372/332; SO4 16/14/12/10 -> 355/379/359/300; SO6 16/14/12 -> 255/255/248;
        # SO8 14/12/10 -> 219/224/188; heat R = 1 16/12/10/8... -> 575/497/676 (two CTAs per SM)
        if wave:
            return {1: 12, 2: 14, 3: 16, 4: 12}[R]
        return 10 if R == 1 else 16
    if not wave and TK == 4 and R <= 2:
        return 8
    return None


def _static_ring(ndim: int, wave: int, R: int) -> bool:
    """Untiled 3-D instances built as sweep1s_kernel (ring of exactly 2r+1 slots, compile-time
    slot/queue indices): where 2r+1 slots leave >= 5 planes of prefetch and, with the cp.async
    staging, fit in shared memory (Geom1S::OK) -- and where it measured faster (C5 SO12: 285.5 vs
    274.4 GPts/s)."""
    # R = 8 (staging depth 3): equal to sweep1 with per-axis weights (241 / 241), +3.4 % with the
    # isotropic-weight instance (C4 254.3 vs 245.9 GPts/s, same-box A/B)
    return ndim == 3 and R in (5, 6, 8)


def _exch(wave: int, R: int) -> bool:
    """T_k = 2 instances built as the two-role exchange pass (sweepx.cuh): wave r >= 3 (measured
    faster than the overlapped-tile sweep2 at SO8 and SO12; heat C2 measured 276 GPts/s vs 486 for
    sweep2, so heat keeps sweep2 -- DESIGN.md §10)."""
    return bool(wave) and R >= 3


# T_k -> (rows per warp, warps) of sweeph (kind 5): regions of 68 / 70 / 72 rows keep a 64-row output
# tile (256 and 512 split into whole tiles); measured same box vs 64-row regions (4 x 16), GPts/s:
# C2 T_k=2/3/4 904/980/1017 vs 780/873/878; 512^3 1176/1169/1205 vs 1186/1224/1094
HEAT_H = {2: (4, 17), 3: (5, 14), 4: (6, 12)}


def _heat_h(R: int, TK: int) -> bool:
    """Heat T_k > 1 instances built as sweeph (kind 5: every level in one warp's registers, x
    neighbours by SHFL, one CTA barrier per step; DESIGN.md §6 G5)."""
    return R == 1 and TK in (2, 3, 4)


def instances():
    """(ndim, wave, R, TK, VY, NWY, kind) compiled into this build.
    For kind 2 the NWY slot holds the output rows OY of the instance."""
    out = []
    for wave in (0, 1):
        for R in range(1, 9):
            ncw, vy = _t1_geom(3, wave, R)
            out.append((3, wave, R, 1, vy, ncw, 3 if _static_ring(3, wave, R) else 1))
            oy = _sweep2_oy(wave, R, 2)
            if not wave and _heat_h(R, 2):
                out.append((3, 0, R, 2) + HEAT_H[2] + (5,))
            elif _exch(wave, R):
                out.append((3, wave, R, 2, vy, ncw, 4))        # L1/L2 roles, untiled geometry
            elif oy:
                out.append((3, wave, R, 2, 2, oy, 2))
            else:
                out.append((3, wave, R, 2) + _vy_nwy(3, R, 2) + (0,))
        for R in range(1, 9):
            ncw, vy = _t1_geom(2, wave, R)
            out.append((2, wave, R, 1, vy, ncw, 1))
        out.append((2, wave, 1, 2) + _vy_nwy(2, 1, 2) + (0,))
        out.append((2, wave, 1, 4) + _vy_nwy(2, 1, 4) + (0,))
    # heat T_k = 4 (sweep2); T_k = 8 (first-generation kernel, 46 GPts/s on 512^3 vs 708 at T = 1)
    # is retired: stencil_create reports ST_EUNSUPPORTED for it
    out.append((3, 0, 1, 3) + HEAT_H[3] + (5,))
    for R, TK in ((1, 4), (2, 4)):
        if _heat_h(R, TK):
            out.append((3, 0, R, TK) + HEAT_H[TK] + (5,))
            continue
        oy = _sweep2_oy(0, R, TK)
        out.append((3, 0, R, TK, 2, oy, 2) if oy else (3, 0, R, TK) + _vy_nwy(3, R, TK) + (0,))
    return out


def _gen_sources(groups: int, inst=None, outdir: str = BUILD):
    os.makedirs(outdir, exist_ok=True)
    inst = instances() if inst is None else inst
    groups = max(1, min(groups, len(inst)))
    files = []
    per = [inst[i::groups] for i in range(groups)]
    for gi, group in enumerate(per):
        lines = ['#include "registry.h"', "namespace st {", f"extern const KernelEntry kInst{gi}[] = {{"]
        for (ndim, wave, R, TK, VY, NWY, kind) in group:
            w = 'true' if wave else 'false'
            if kind == 1:
                lines.append(f"  make_entry1<{R}, {w}, {ndim}, {NWY}, {VY}>(),")
            elif kind == 3:
                lines.append(f"  make_entry1s<{R}, {w}, {NWY}, {VY}>(),")
            elif kind == 2:
                lines.append(f"  make_entry2<{R}, {TK}, {w}, {NWY}>(),")   # NWY = output rows
            elif kind == 4:
                lines.append(f"  make_entryX<{R}, {w}, {NWY}, {VY}>(),")
            elif kind == 5:
                lines.append(f"  make_entryH<{R}, {TK}, {VY}, {NWY}>(),")
            else:
                lines.append(f"  make_entry<{R}, {TK}, {w}, {ndim}, {VY}, {NWY}>(),")
        lines += ["};", f"extern const int kInst{gi}Count = {len(group)};", "}  // namespace st", ""]
        files.append((os.path.join(outdir, f"inst_{gi}.cu"), "\n".join(lines)))
    reg = ['#include "registry.h"', "#include <vector>", "namespace st {"]
    for gi in range(groups):
        reg.append(f"extern const KernelEntry kInst{gi}[]; extern const int kInst{gi}Count;")
    reg.append("static std::vector<KernelEntry> build_all() {\n  std::vector<KernelEntry> v;")
    for gi in range(groups):
        reg.append(f"  v.insert(v.end(), kInst{gi}, kInst{gi} + kInst{gi}Count);")
    reg.append("  return v;\n}")
    reg.append("static const std::vector<KernelEntry>& all() { static const std::vector<KernelEntry> v = build_all(); return v; }")
    reg.append("const KernelEntry* registry_begin() { return all().data(); }")
    reg.append("const KernelEntry* registry_end() { return all().data() + all().size(); }")
    reg.append("const KernelEntry* find_kernel(int ndim, int time_order, int radius, int tk) {\n"
               "  for (const auto& e : all())\n"
               "    if (e.ndim == ndim && e.time_order == time_order && e.radius == radius && e.tk == tk) return &e;\n"
               "  return nullptr;\n}")
    reg += ["}  // namespace st", ""]
    files.append((os.path.join(outdir, "registry.cu"), "\n".join(reg)))
    for path, text in files:
        if not os.path.exists(path) or open(path).read() != text:
            with open(path, "w") as f:
                f.write(text)
    return [f for f, _ in files]


def _digest(paths, extra=()):
    h = hashlib.sha256()
    for pth in sorted(paths):
        with open(pth, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS + list(extra)).encode())
    return h.hexdigest()[:16]


def _compile(src: str, outdir: str = BUILD, defines=()):
    obj = os.path.join(outdir, os.path.basename(src) + ".o")
    # every header of csrc/ and the ABI header: any edit rebuilds every object that may include it
    deps = [src] + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) \
        + [os.path.join(HERE, "..", "include", "stencil.h")]
    stamp = obj + ".stamp"
    d = _digest(deps, defines)
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == d:
        return obj, ""
    cmd = [NVCC] + ARCH + FLAGS + list(defines) + ["-I", CSRC, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    with open(stamp, "w") as f:
        f.write(d)
    return obj, r.stderr


def _build(outdir, lib, inst=None, defines=(), groups=12, jobs=0, verbose=False):
    srcs = _gen_sources(groups, inst, outdir) + [os.path.join(CSRC, "abi.cu")]
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    objs, logs = [], []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for obj, log in ex.map(lambda s: _compile(s, outdir, defines), srcs):
            objs.append(obj)
            logs.append(log)
    if verbose:
        with open(os.path.join(outdir, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    need = not os.path.exists(lib) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs)
    if need:
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return lib


def build(force: bool = False, jobs: int = 0, verbose: bool = False) -> str:
    if force and os.path.isdir(BUILD):
        for f in os.listdir(BUILD):
            if f.endswith(".o") or f.endswith(".stamp"):
                os.remove(os.path.join(BUILD, f))
    return _build(BUILD, LIB, jobs=jobs, verbose=verbose)


def build_variant(name: str, defines=(), only=None, t1=None, verbose: bool = True,
                  static_r=None, oy2=None, heat_h=None) -> str:
    """Experimental library _variants/libstencil_<name>.so with extra -D flags and (optionally)
    only the instances whose (ndim, wave, R, TK) is listed; load it with ST_LIB=<path>."""
    inst = instances()
    if only is not None:
        inst = [i for i in inst if tuple(i[:4]) in set(map(tuple, only))]
    outdir = os.path.join(HERE, "_variants", name)
    os.makedirs(os.path.join(HERE, "_varlib"), exist_ok=True)
    lib = os.path.join(HERE, "_varlib", f"libstencil_{name}.so")   # shipped to the GPU box
    if oy2 is not None:        # {(wave, R, TK): OY} output rows of time-tiled (kind 2) instances
        inst = [i[:5] + (oy2.get((i[1], i[2], i[3]), i[5]),) + i[6:] if i[6] == 2 else i for i in inst]
    if static_r is not None:   # radii whose 3-D untiled instances use the static ring (kind 3)
        inst = [i[:6] + ((3 if i[2] in static_r else 1),) if i[0] == 3 and i[3] == 1 and i[6] in (1, 3)
                else i for i in inst]
    if heat_h is not None:   # {T_k: (rows per warp, warps)} of the heat time-tiled kernel (kind 5)
        inst = [i[:4] + heat_h.get(i[3], (i[4], i[5])) + i[6:] if i[6] == 5 else i for i in inst]
    if t1 is not None:   # (consumer warps, rows per warp) of the untiled kernel
        inst = [i[:4] + (t1[1], t1[0], i[6]) if i[6] in (1, 3) else i for i in inst]
    return _build(outdir, lib, inst, list(defines), groups=4, verbose=verbose)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=0)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=a.v))
