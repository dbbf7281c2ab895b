"""Compare the register-window LU against the generic LU (factor pools, row-major
copies, reciprocal diagonals) on small shapes; run on the GPU box."""
import ctypes as C, os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_1811_03559_b200 as spk
    from oracle.oracle import Oracle
    n, k, p = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    o = Oracle()
    band = o.generate_band(5, n, k, k, 1.5)
    a = spk.BandedMatrix(n, k, k, band)
    plan = spk.gpu_plan(n, k, k, 1, False, p)
    f = spk.factorize(a, plan)
    L = spk.lib()
    L.spk_fact_dump.restype = C.c_int64
    L.spk_fact_dump.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    out = {}
    for w in range(3):
        sz = L.spk_fact_dump(f._h, w, None)
        buf = np.zeros(sz)
        L.spk_fact_dump(f._h, w, buf.ctypes.data)
        out[w] = buf.tolist()
    print(json.dumps(out))
    sys.exit(0)

for (n, k, p) in [(64, 1, 2), (64, 1, 4), (512, 4, 4), (300, 16, 3), (2000, 40, 4)]:
    res = {}
    for gen in ("0", "1"):
        env = dict(os.environ, SPK_GENERIC=gen)
        r = subprocess.run([sys.executable, __file__, "child", str(n), str(k), str(p)], env=env,
                           capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-2000:])
        res[gen] = json.loads(r.stdout.strip().splitlines()[-1])
    for w, name in enumerate(["fac", "tfac", "dinv"]):
        x, y = np.array(res["0"][str(w)]), np.array(res["1"][str(w)])
        d = np.abs(x - y)
        bad = np.nonzero(d > 1e-12 * max(1, np.abs(y).max()))[0]
        print(n, k, p, name, "size", x.size, "max diff", d.max() if d.size else 0, "nbad", bad.size, "first", bad[:12].tolist(),
              "fast", x[bad[:6]].tolist(), "gen", y[bad[:6]].tolist())
