"""Build (here) / time (on the box) variants of the TMA-staged FULL_FD kernel
(cm_tma.cuh, k_collide_stream_fd_tma) at 512^3, fp64 and fp32 storage.

  python scripts/fd_tma_variants.py build
  python scripts/fd_tma_variants.py run      # bench.py --corrections full_fd per variant
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "varbuild")  # git-ignored, travels to the GPU box
# The EARLY / MAXNREG / SHAPE / RING3 / PF switches below belonged to experiments whose kernel code
# was removed after measuring them slower (profiles/r2/fd_tma_variants.jsonl);
# with the current sources they are no-ops.
VARIANTS = {
    "base": ["LBM_FD_TMA_EARLY=0"],
    "shape": ["LBM_FD_TMA_SHAPE=1"],
    "ring3": ["LBM_FD_TMA_RING3=1"],
    "pf1": ["LBM_FD_TMA_PF=1"],
    "pf2": ["LBM_FD_TMA_PF=2"],
    "pf4": ["LBM_FD_TMA_PF=4"],
    "early": ["LBM_FD_TMA_EARLY=1"],
    "early_m32_2": ["LBM_FD_TMA_EARLY=1", "LBM_FD_TMA_MINB32=2"],
    "early_r200": ["LBM_FD_TMA_EARLY=1", "LBM_FD_TMA_MAXNREG=1"],
    "base_r200": ["LBM_FD_TMA_EARLY=0", "LBM_FD_TMA_MAXNREG=1"],
}

if sys.argv[1] == "build":
    from paper_2107_14774_b200 import build as B
    os.makedirs(VDIR, exist_ok=True)
    only = sys.argv[2:] or list(VARIANTS)
    for n in only:
        out = os.path.join(VDIR, f"lib_fdtma_{n}.so")
        B.build(out=out, defines=VARIANTS[n])
        log = open(out + ".ptxas.log").read()
        for t in ("d", "f"):
            m = re.search(r"k_collide_stream_fd_tmaI" + t + r"Li1EE.*?\n.*?(\d+) bytes spill stores.*?\n.*?Used (\d+) registers",
                          log, re.S)
            print(n, t, "spill", m.group(1) if m else "?", "regs", m.group(2) if m else "?", flush=True)
else:
    only = sys.argv[2:] or list(VARIANTS)
    for n in only:
        for prec in ("fp64", "fp32"):
            env = dict(os.environ, LBM_CUBOID_LIB=os.path.join(VDIR, f"lib_fdtma_{n}.so"), LBM_FD_TMA="1")
            extra = os.environ.get("FD_VARIANT_ARGS", "").split()
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3",
                                "--corrections", "full_fd", "--precision", prec, "--no-e2e", "--no-cpu-baseline",
                                *extra],
                               capture_output=True, text=True, env=env, timeout=400)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                print(json.dumps({"variant": n, "precision": prec, "mlups": round(d["value"]),
                                  "ms_per_step": d["ms_per_step"], "frac": d["roofline"]["frac"],
                                  "kernel": d["roofline"]["kernel"], "clocks": d["clocks"]}), flush=True)
            except Exception:  # noqa: BLE001
                print(n, prec, "FAILED", r.stderr[-1500:], flush=True)
