"""Overlap of the halo with the interior on one B200 (SURVEY §5 "nsys for
overlap"; nsys is not installed here, so the library's event trace,
lbm_cuboid_trace, stands in): config-5 weak slab (512^3, periodic TGV) with the
multi-GPU step structure forced on one GPU, NCCL halo (send to self) and the
fused P2P halo (this slab its own neighbour).  Per step: start/end of the
boundary-plane launch, the NCCL exchange, and the interior launch on their
streams; reported: how much of the boundary launch and of the halo exchange
lies inside the interior launch's interval.

  python scripts/overlap_trace.py [steps] > profiles/r2/overlap_trace.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def overlap(a, b):
    lo, hi = max(a[0], b[0]), min(a[1], b[1])
    return max(0.0, hi - lo)


def run(halo, steps):
    import paper_2107_14774_b200 as P
    import synth

    w = synth.CONFIGS["weak"]
    kw = dict(w.params(), device=0)
    if halo == "nccl":
        g = P.Lattice(**kw, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id())
    else:
        g = P.Lattice(**kw, halo=P.HALO_P2P)
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0)
    g.init_fields(rho, u)
    g.step(3)
    g.trace(True)
    g.step(steps)
    rows = g.trace_read()
    g.trace(False)
    g.close()
    # group per step: [boundary, (nccl), interior]
    per = []
    bnd = [r for r in rows if r["kind"] == "boundary"]
    inter = [r for r in rows if r["kind"] == "collide"]
    halo_rows = [r for r in rows if r["kind"] == "nccl_halo"]
    for k in range(min(len(bnd), len(inter))):
        b, i = bnd[k], inter[k]
        rec = {"boundary_ms": [b["t0_ms"], b["t1_ms"]], "boundary_stream": b["stream"],
               "interior_ms": [i["t0_ms"], i["t1_ms"]],
               "boundary_inside_interior": overlap((b["t0_ms"], b["t1_ms"]), (i["t0_ms"], i["t1_ms"])) /
               max(b["t1_ms"] - b["t0_ms"], 1e-9)}
        if k < len(halo_rows):
            hh = halo_rows[k]
            rec["halo_ms"] = [hh["t0_ms"], hh["t1_ms"]]
            rec["halo_inside_interior"] = overlap((hh["t0_ms"], hh["t1_ms"]), (i["t0_ms"], i["t1_ms"])) / max(
                hh["t1_ms"] - hh["t0_ms"], 1e-9)
        per.append(rec)
    return {"halo": halo, "steps": per, "rows": rows}


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    out = {"what": "event trace of the multi-GPU step structure on one B200 (512^3 slab, fp64)",
           "runs": [run("nccl", steps), run("p2p", steps)]}
    print(json.dumps(out, indent=1))
