"""Probe the TMA collide-stream kernel variants (one subprocess per variant and
case, so a faulting variant cannot poison the next): create, init, 3 steps,
sync, compare with the one-node-per-thread kernel."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {
    "tgv256_fp64": dict(w="tgv", nx=256, ny=9, nz=6, precision=0),
    "tgv256_fp32": dict(w="tgv", nx=256, ny=9, nz=6, precision=1),
    "cavity136_fp64": dict(w="cavity100", nx=136, ny=10, nz=6, precision=0),
}


def child(case):
    sys.path.insert(0, ROOT)
    import numpy as np

    import paper_2107_14774_b200 as P
    import synth

    d = dict(CASES[case])
    w = synth.CONFIGS[d.pop("w")].scaled(**d)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 3)
    out = {}
    for tma in ("0", "1"):
        os.environ["LBM_TMA"] = tma
        g = P.Lattice(**w.params(), graphs=1)
        g.init_fields(rho, u)
        g.step(3)
        g.sync()
        out[tma] = g.get_populations()
        g.close()
    print(json.dumps({"case": case, "maxdiff": float(np.abs(out["0"] - out["1"]).max())}))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(sys.argv[2])
        sys.exit(0)
    libs = sys.argv[1:] or ["paper_2107_14774_b200/liblbm_cuboid.so"]
    for lib in libs:
        for case in CASES:
            env = dict(os.environ, LBM_CUBOID_LIB=os.path.join(ROOT, lib))
            try:
                r = subprocess.run([sys.executable, __file__, "child", case], env=env, capture_output=True, text=True,
                                   timeout=120)
                tail = (r.stdout.strip().splitlines() or [""])[-1]
                err = "" if r.returncode == 0 else r.stderr.strip().splitlines()[-1][:200]
                print(f"{lib} {case} rc={r.returncode} {tail} {err}", flush=True)
            except subprocess.TimeoutExpired:
                print(f"{lib} {case} TIMEOUT", flush=True)
