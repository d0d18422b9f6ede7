"""Build (here) / time (on the box) variants of the fused FULL_FD kernel.

  python scripts/fd_variants.py build
  python scripts/fd_variants.py run      # bench.py --corrections full_fd per variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "fd_variants")
VARIANTS = {  # tile / chunk shapes of the fused FULL_FD kernel
    "zc32_ty4": ["LBM_FD_ZC=32", "LBM_FD_TY=4", "LBM_FD_MINB=4"],
    "zc16_ty4": ["LBM_FD_ZC=16", "LBM_FD_TY=4", "LBM_FD_MINB=4"],
    "zc64_ty4": ["LBM_FD_ZC=64", "LBM_FD_TY=4", "LBM_FD_MINB=4"],
    "zc32_ty8": ["LBM_FD_ZC=32", "LBM_FD_TY=8", "LBM_FD_MINB=2"],
    "zc32_tx64_ty4": ["LBM_FD_ZC=32", "LBM_FD_TX=64", "LBM_FD_TY=4", "LBM_FD_MINB=2"],
}

if sys.argv[1] == "build":
    from paper_2107_14774_b200 import build as B
    import re
    os.makedirs(VDIR, exist_ok=True)
    for n, d in VARIANTS.items():
        out = os.path.join(VDIR, f"lib_{n}.so")
        B.build(out=out, defines=d)
        log = open(out + ".ptxas.log").read()
        m = re.search(r"k_collide_stream_fdIdLi1EE.*?\n.*?(\d+) bytes spill stores.*?\n.*?Used (\d+) registers", log, re.S)
        print(n, "spill", m.group(1) if m else "?", "regs", m.group(2) if m else "?")
else:
    for n in VARIANTS:
        env = dict(os.environ, LBM_CUBOID_LIB=os.path.join(VDIR, f"lib_{n}.so"), LBM_FD_FUSED="1")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3",
                            "--corrections", "full_fd", "--no-e2e", "--no-cpu-baseline"],
                           capture_output=True, text=True, env=env, timeout=300)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(json.dumps({"variant": n, "mlups": d["value"], "ms_per_step": d["ms_per_step"],
                              "clocks": d["clocks"]}), flush=True)
        except Exception:  # noqa: BLE001
            print(n, "FAILED", r.stderr[-1500:], flush=True)
