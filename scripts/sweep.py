#!/usr/bin/env python
"""Kernel-variant sweep on one GPU (run under gpurun).

  python scripts/sweep.py build          # here: compile variants into build/variants/
  python scripts/sweep.py run [names]    # on the box: time each variant in a subprocess

Each variant times the bench workload (config 5 weak, 512^3, fp64 unless the
variant says fp32): back-to-back steps (one event pair), per-step events, and
steps separated by idle gaps; nvidia-smi samples clocks/power meanwhile.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "variants")

VARIANTS = {
    "base": [],
    "b128m5": ["LBM_MINB=5"],
    "b128m6": ["LBM_MINB=6"],
    "b128m7": ["LBM_MINB=7"],
    "b128m8": ["LBM_MINB=8"],
    "b64m12": ["LBM_BLOCK=64", "LBM_MINB=12"],
    "b64m14": ["LBM_BLOCK=64", "LBM_MINB=14"],
    "b64": ["LBM_BLOCK=64"],
    "b256": ["LBM_BLOCK=256"],
    "b256m3": ["LBM_BLOCK=256", "LBM_MINB=3"],
    "ld1": ["LBM_LDMODE=1"],
    "st1": ["LBM_STMODE=1"],
    "debug": ["LBM_DEBUG_BOUNDS=1"],
}


def build(names):
    from paper_2107_14774_b200 import build as B

    os.makedirs(VDIR, exist_ok=True)
    for n in names:
        out = os.path.join(VDIR, f"lib_{n}.so")
        B.build(out=out, defines=VARIANTS[n])
        log = open(out + ".ptxas.log").read()
        import re

        regs = re.findall(r"k_collide_stream.*?\n.*?\n.*?Used (\d+) registers", log, re.S)
        spills = re.findall(r"k_collide_stream.*?\n.*?(\d+) bytes spill stores", log, re.S)
        print(n, "regs", regs, "spill", spills)


def child(name, prec, nzl):
    import numpy as np
    import torch

    import paper_2107_14774_b200 as P
    import synth

    w = synth.CONFIGS["weak"].scaled(nz=nzl, precision=prec)
    lat = P.Lattice(device=0, **w.params())
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device="cuda")
    lat.init_fields(rho, u)
    del rho, u
    s = lat.stream
    lat.step(5)
    torch.cuda.synchronize()
    res = {"variant": name, "prec": prec, "nodes": w.nodes}
    # (a) back-to-back, one event pair
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 40
    a.record(s)
    lat.step(n)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    res["b2b_ms"] = ms
    res["b2b_mlups"] = w.nodes / ms / 1e3
    # (b) per-step events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for e0, e1 in ev:
        e0.record(s)
        lat.step(1)
        e1.record(s)
    torch.cuda.synchronize()
    t = [e0.elapsed_time(e1) for e0, e1 in ev]
    res["per_step_ms"] = [float(np.mean(t)), float(np.min(t)), float(np.max(t)), t[0], t[-1]]
    # (c) host sync (no sleep) / 1 ms / 30 ms idle gaps between steps
    for label, gap in (("sync_ms", 0.0), ("gap1_ms", 0.001), ("gap30_ms", 0.03)):
        tg = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            lat.step(1)
            e1.record(s)
            torch.cuda.synchronize()
            tg.append(e0.elapsed_time(e1))
            if gap:
                time.sleep(gap)
        res[label] = [float(np.mean(tg)), float(np.min(tg))]
    # (d) a long back-to-back run: 10 blocks of 20 steps
    blk = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        lat.step(20)
        e1.record(s)
        blk.append((e0, e1))
    torch.cuda.synchronize()
    res["long_b2b_ms"] = [round(a.elapsed_time(b) / 20, 4) for a, b in blk]
    res["bad"] = lat.check(raise_on_unstable=False)["bad_nodes"]
    print("RESULT " + json.dumps(res), flush=True)


def run(names, prec=0, nzl=512):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                            "power.draw.instant,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "50"],
                           stdout=open(os.path.join(ROOT, "gpurun_out", f"sweep_smi_{prec}.csv"), "w"))
    try:
        for n in names:
            env = dict(os.environ, LBM_CUBOID_LIB=os.path.join(VDIR, f"lib_{n}.so"))
            t0 = time.time()
            r = subprocess.run([sys.executable, __file__, "child", n, str(prec), str(nzl)], env=env,
                               capture_output=True, text=True, timeout=600)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
            print(line[0][7:] if line else f"{n} FAILED rc={r.returncode} {r.stderr[-800:]}", flush=True)
            print(f"  ({n}: {time.time() - t0:.1f} s)", flush=True)
    finally:
        smi.terminate()


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        build(sys.argv[2:] or list(VARIANTS))
    elif cmd == "run":
        prec = int(os.environ.get("PREC", "0"))
        run(sys.argv[2:] or list(VARIANTS), prec=prec, nzl=int(os.environ.get("NZL", "512")))
    elif cmd == "child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
