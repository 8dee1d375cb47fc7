"""Per-launch HBM figures of an `ncu --set full` capture of a sweep kernel.

    python tools/ncu_report.py REP.ncu-rep --key C5_tk1 --points 452984832 --steps 1 [--alg 20]

Prints one JSON object: kernel, duration, dram bytes read/written per launch, effective DRAM bytes
per interior point update (= dram bytes / (points x time levels the launch advances)), achieved
DRAM GB/s (= dram bytes / ncu duration) as a fraction of the nominal 8 TB/s and of the measured copy
bandwidth (MEASURED_PEAKS.json), and the algorithmic bytes per update for comparison.  With
--merge it also records dram_bytes_per_launch under KEY in profiles/ncu_traffic.json (read by
bench.py for the roofline "traffic" field).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [dict(zip(h, r)) for r in rows[2:]], dict(zip(h, u))


def num(s):
    return float(str(s).replace(",", ""))


def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return v * f


def to_seconds(v, unit):
    return v * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                "nsecond": 1e-9, "s": 1.0, "second": 1.0}[unit]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--key", required=True)
    ap.add_argument("--points", type=float, required=True, help="interior points per launch")
    ap.add_argument("--steps", type=int, default=1, help="time levels one launch advances")
    ap.add_argument("--alg", type=float, default=None, help="algorithmic bytes per point per launch")
    ap.add_argument("--merge", action="store_true")
    a = ap.parse_args()
    rows, units = raw(a.rep)
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    out = []
    for r in rows:
        rd = to_bytes(num(r["dram__bytes_read.sum"]), units["dram__bytes_read.sum"])
        wr = to_bytes(num(r["dram__bytes_write.sum"]), units["dram__bytes_write.sum"])
        t = to_seconds(num(r["gpu__time_duration.sum"]), units["gpu__time_duration.sum"])
        upd = a.points * a.steps
        gbs = (rd + wr) / t / 1e9
        d = {"key": a.key, "kernel": r.get("Kernel Name", "?")[:80], "duration_ms": round(t * 1e3, 4),
             "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
             "dram_bytes_per_update": round((rd + wr) / upd, 3),
             "alg_bytes_per_update": None if a.alg is None else round(a.alg / a.steps, 3),
             "dram_gbs": round(gbs, 1), "frac_of_8TBs": round(gbs / 8000, 4),
             "frac_of_measured_copy": round(gbs / peak, 4),
             "dram_throughput_pct_ncu": num(r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
             "gpts_per_s_under_ncu": round(upd / t / 1e9, 1),
             "registers": int(num(r["launch__registers_per_thread"])),
             "grid": r.get("launch__grid_size"), "block": r.get("launch__block_size")}
        out.append(d)
        print(json.dumps(d))
    if a.merge and out:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        db = json.load(open(path)) if os.path.exists(path) else {}
        db[a.key] = out[-1]
        with open(path, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
