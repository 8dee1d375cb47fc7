"""Compare full-grid runs of different libraries / t_kernel on one config (debug helper)."""
import hashlib, os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))

def child(cfg, nt, tk):
    import numpy as np
    import workloads as W
    from harness import gpu_run
    p = W.problem(cfg)
    out = gpu_run(p, nt=nt, t_kernel=tk)
    res = {}
    for name, a in zip(("P", "C", "T"), out):
        res[name] = hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]
    np.save(f"/tmp/cmp_{os.environ.get('TAG','x')}_C.npy", out[1])
    print("RESULT", json.dumps(res))

if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4])); sys.exit(0)
    cfg, nt = sys.argv[1], sys.argv[2]
    libs = sys.argv[3].split(",") if len(sys.argv) > 3 else []
    runs = [("main_tk2", None, 2), ("main_a", None, 1), ("main_b", None, 1), ("main_c", None, 1)]
    for v in libs:
        for rep in ("a", "b"):
            runs.append((f"{v}_{rep}", f"paper_1707_02347_b200/_varlib/libstencil_{v}.so", 1))
    for tag, lib, tk in runs:
        env = dict(os.environ, TAG=tag)
        if lib: env["ST_LIB"] = lib
        r = subprocess.run([sys.executable, __file__, "child", cfg, nt, str(tk)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        print(tag, line[0][7:] if line else r.stderr[-500:], flush=True)
    import numpy as np
    a = np.load("/tmp/cmp_main_tk2_C.npy")
    for tag, _, _ in runs[1:]:
        b = np.load(f"/tmp/cmp_{tag}_C.npy")
        d = np.argwhere(a != b)
        print(tag, "ndiff vs main_tk2", len(d), "first", d[:2].tolist())
