#!/usr/bin/env python
"""Benchmark of the fused D3Q27 cuboid central-moment collide-stream (fp64).

  python bench.py --gpus N --steps K --warmup W [--impl cuda|reference]
  (N > 1: launched by torchrun, one rank per GPU, NCCL)

Workload (BASELINE.json configs[4], config 5 weak): periodic Taylor-Green vortex,
512 x 512 x 512 nodes PER GPU (global 512 x 512 x 512N, z-slab decomposition),
r = 1, s = 2, nu = 0.01, omega_xi = omega_1 = omega_high = 1, FULL_LOCAL
corrections, fp64.  One step = one pull-stream + collide of every node.
Metric: MLUPS (10^6 lattice-node updates per second), whole job.

`value` is device-timed (CUDA events on the library's compute stream, max over
ranks, inputs resident in HBM; the 58 GB per-GPU working set per step is far
larger than the 126 MB L2, so no flush is needed; for the small configs, whose
population buffers fit in L2, every timed step is preceded by an untimed write
of a 512 MB buffer that flushes L2, and `value` sums per-step event timings).  `e2e` is the same metric
through the public C ABI with HOST buffers: host->device copy of the initial
fields, K steps, device->host copy of rho and u, all inside the timed region.
"""
from __future__ import annotations

import argparse
import glob
import hashlib
import stat
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
L2_BYTES = 126 << 20       # B200 L2
FLUSH_BYTES = 512 << 20    # written between timed steps when the buffers fit in L2
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "D3Q27 cuboid CM-LBM MLUPS (fp64) at 1/2/4/8 B200; achieved roofline fraction"
# the one bounded oracle sample both CPU legs time (cpu_baseline and --impl reference)
ORACLE_SAMPLE = (48, 48, 24)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--workload", default="weak", choices=["weak", "strong", "shear", "cavity100", "cavity1000", "tgv", "duct"])
    ap.add_argument("--streaming", choices=["ab", "aa"], default="ab",
                    help="aa: one population buffer updated in place (single GPU)")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nz-per-gpu", type=int, default=None, help="override the per-GPU slab depth")
    ap.add_argument("--corrections", choices=["full_local", "low_mach", "off", "full_fd", "full_fd_lag"],
                    default="full_local")
    ap.add_argument("--model", choices=["cm", "rm"], default="cm")
    ap.add_argument("--halo", choices=["auto", "nccl", "p2p"], default="auto",
                    help="nccl: force the multi-GPU step structure (boundary launch, NCCL ghost-plane "
                         "exchange on the comm stream, interior launch) even on one GPU (send to self); "
                         "p2p: fused halo (the boundary-plane kernel stores into the neighbours' ghost "
                         "planes over peer memory, concurrent with the interior; on one GPU into its own)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: print this rank's plan (slab, workload, launches) and, under torchrun, "
                         "check the max-over-ranks aggregation over a gloo process group")
    return ap.parse_args()


def workload(args, world):
    w = synth.CONFIGS[args.workload]
    if args.precision == "fp32":
        w = w.scaled(precision=synth.PREC_FP32)
    corr = {"full_local": synth.CORR_FULL_LOCAL, "low_mach": synth.CORR_LOW_MACH, "off": synth.CORR_OFF,
            "full_fd": synth.CORR_FULL_FD, "full_fd_lag": synth.CORR_FULL_FD_LAG}[args.corrections]
    w = w.scaled(corrections=corr, model=synth.MODEL_RM if args.model == "rm" else synth.MODEL_CM)
    nzl = args.nz_per_gpu or w.nz
    if args.workload == "weak":
        w = w.scaled(nz=nzl * world)      # weak scaling: fixed 512^3 per GPU
    elif w.nz % world:
        raise SystemExit(f"nz={w.nz} not divisible by {world} GPUs")
    return w


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """`nvidia-smi -lms 100` running DURING the timed region (started before,
    terminated after): median SM clock under load and throttle reasons seen."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, log_path=None):
        self.index = index
        self.log_path = log_path
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=10)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()
            if self.log_path:
                with open(self.log_path, "w") as fh:
                    fh.write(self.out)

    def summary(self):
        rows = [[c.strip() for c in ln.split(",")] for ln in self.out.splitlines() if ln.count(",") >= 6]

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        pw = [num(r[2]) for r in rows]
        load = [r for r, p in zip(rows, pw) if p is not None and p > 350.0] or rows
        sm = [num(r[0]) for r in load if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max(p for p in pw if p is not None) if any(p is not None for p in pw) else None}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def kernel_source_hash():
    """sha256 (16 hex digits) of the CUDA sources and the ABI header: the key that
    ties a committed ncu traffic measurement to the build it was taken on."""
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2107_14774_b200", "csrc", "*.cu*")))
    files.append(os.path.join(ROOT, "include", "lbm_cuboid.h"))
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(workload_name, precision, kernel, nodes_per_launch):
    """dram bytes (read + write) per launch of the collide-stream kernel from a
    committed ncu capture (profiles/ncu_traffic.json, written by
    scripts/ncu_traffic_update.py) of THIS build (kernel source hash), workload,
    precision, kernel and launch size; None if no capture matches."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, "no profiles/ncu_traffic.json"
    with open(path) as fh:
        entries = json.load(fh).get("entries", [])
    src = kernel_source_hash()
    for e in entries:
        if (e.get("workload"), e.get("precision"), e.get("kernel"), int(e.get("nodes_per_launch", -1)),
                e.get("source_hash")) == (workload_name, precision, kernel, int(nodes_per_launch), src):
            return e["dram_bytes_per_launch"], e.get("source", "")
    return None, f"no ncu capture of this build (kernel sources {src}) for this workload/kernel/launch size"


# --------------------------------------------------------------- cpu oracle
def host_cpu():
    """(CPU model, logical cores) of this host, for the cpu_baseline record."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


class pinned_to_one_core:
    """Run the single-threaded oracle pinned to one host core."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.core = max(self.prev)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.prev)


def oracle_mlups(w, budget_s=15.0, grid=ORACLE_SAMPLE, max_steps=None):
    """The CPU oracle as it stands (single thread, pinned to one core), on a
    bounded sample of the workload: same physics on a smaller grid, as many
    steps as fit in budget_s."""
    import oracle as O

    nx, ny, nz = grid
    ws = w.scaled(nx=nx, ny=ny, nz=nz)
    o = O.Oracle(**ws.params())
    rho, u = synth.initial_fields(ws)
    o.init_fields(rho, u)
    with pinned_to_one_core():
        t0 = time.perf_counter()
        n = 0
        while True:
            o.step(1)
            n += 1
            el = time.perf_counter() - t0
            if el >= budget_s or (max_steps and n >= max_steps):
                break
    return ws.nodes * n / el / 1e6, n, ws


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = args.gpus
    w = workload(args, world)
    steps, warm = args.steps, args.warmup
    import oracle as O

    ws = w.scaled(nx=ORACLE_SAMPLE[0], ny=ORACLE_SAMPLE[1], nz=ORACLE_SAMPLE[2])
    o = O.Oracle(**ws.params())
    rho, u = synth.initial_fields(ws)
    o.init_fields(rho, u)
    with pinned_to_one_core():
        for _ in range(warm):
            o.step(1)
        t0 = time.perf_counter()
        for _ in range(steps):
            o.step(1)
        el = time.perf_counter() - t0
    v = ws.nodes * steps / el / 1e6
    sample = f"oracle on {ws.nx}x{ws.ny}x{ws.nz} (same physics as {w.name}), {steps} steps, 1 thread pinned to 1 core"
    line = {"metric": METRIC, "value": v, "unit": "MLUPS", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": el / steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": w.name, "nodes_global": w.nodes, "sample": sample},
            "cpu_baseline": {"value": v, "unit": "MLUPS", "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu_model": host_cpu()[0], "host_logical_cores": host_cpu()[1]},
            "e2e": {"value": v, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- cuda arm
def run_cuda(args):
    import torch
    import torch.distributed as dist

    import paper_2107_14774_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's own INIT lines (rank / nranks of every communicator) for the record: NCCL
        # reads these once, at its first call, which is the torch process group's eager
        # init below.  They go to stderr when that is a pipe or terminal (so rank 0's
        # stdout stays the one JSON line; NCCL would truncate a regular file it reopens),
        # else to stdout, NCCL's default
        if "NCCL_DEBUG" not in os.environ:
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            try:
                if not stat.S_ISREG(os.fstat(2).st_mode):
                    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            except OSError:
                pass
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args, world)
    z0, z1 = synth.slab_range(w.nz, rank, world)
    kw = w.params()
    aa_fit_note = None
    if args.streaming == "ab":
        # two population buffers that do not fit in this GPU's free HBM (config 5 strong,
        # 1024 x 1024 x 512, on one GPU: 2 x 116 GB): the one-buffer AA scheme instead, said so
        from paper_2107_14774_b200 import lbm as _L
        need = 2 * _L.buffer_bytes(_L.make_params(**dict(kw, rank=rank, world=world, device=local)))
        free = torch.cuda.mem_get_info(local)[0]
        if need > 0.95 * free:
            args.streaming = "aa"
            aa_fit_note = (f"AA in place (1 buffer): two buffers ({need / 2**30:.1f} GiB) exceed the "
                           f"free HBM ({free / 2**30:.1f} GiB)")
    if args.streaming == "aa":
        kw["streaming"] = P.STREAM_AA
    if args.halo == "p2p":
        kw["halo"] = P.HALO_P2P
    if world > 1:
        lat = P.distributed_lattice(device=local, **kw)
    elif args.halo == "nccl":
        lat = P.Lattice(device=local, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id(), **kw)
    else:
        lat = P.Lattice(device=local, **kw)
    stream = lat.stream
    nloc = w.nx * w.ny * (z1 - z0)

    def init_device():
        if w.init == "tgv":
            rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, z0, z1, w.nz, xp=torch,
                                      device=torch.device("cuda", local))
        else:
            rh, uh = synth.initial_fields(w, z0, z1, w.nz)
            rho, u = torch.from_numpy(rh).cuda(local), torch.from_numpy(uh).cuda(local)
        lat.init_fields(rho, u)
        torch.cuda.synchronize(local)

    def barrier():
        # drain this rank's GPU work (incl. the library's NCCL halo stream) before
        # the torch collective, so two communicators never have interleaved work in flight
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize(local)

    def max_over_ranks(x):
        if world == 1:
            return x
        torch.cuda.synchronize(local)
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    init_device()
    with torch.cuda.stream(stream):
        lat.step(args.warmup)
    barrier()

    # ---- timed region: exactly K steps between barrier+sync, one event pair on the compute stream
    # (small lattices whose buffers fit in L2: per-step event pairs, L2 flushed before each step)
    flush = None
    if lat.info()["buffer_bytes"] * (1 if args.streaming == "aa" else 2) < 2 * L2_BYTES:
        flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
    l0 = lat.info()["launches"]
    with ClockSampler(local, os.path.join(ROOT, "gpurun_out", f"bench_clocks_rank{rank}.csv")
                      if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None) as clk:
        barrier()
        if flush is None:
            t_start = torch.cuda.Event(enable_timing=True)
            t_end = torch.cuda.Event(enable_timing=True)
            t_start.record(stream)
            lat.step(args.steps)
            t_end.record(stream)
            barrier()
            elapsed = t_start.elapsed_time(t_end)
        else:
            evs = []
            for k in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(k & 0xFF)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                lat.step(1)
                b.record(stream)
                evs.append((a, b))
            barrier()
            elapsed = sum(a.elapsed_time(b) for a, b in evs)
    launches = lat.info()["launches"] - l0
    elapsed_ms = max_over_ranks(elapsed)
    mlups = w.nodes * args.steps / (elapsed_ms * 1e-3) / 1e6
    bpn = lat.info()["bytes_per_node_update"]

    # ---- dominant-kernel duration: the same K steps again with the library's
    # per-launch CUDA events on the compute stream (kept out of the timed region)
    lat.timing(True)
    lat.step(args.steps)
    tk = lat.timing_read()
    lat.timing(False)
    barrier()
    kernel_ms = tk["kernel_ms"] / max(tk["launches"], 1)
    nodes_per_launch = tk["node_updates"] / max(tk["launches"], 1)
    bad = lat.check(raise_on_unstable=False)["bad_nodes"]

    # ---- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        rh = torch.empty((z1 - z0, w.ny, w.nx), dtype=torch.float64, pin_memory=True)
        uh = torch.empty((3, z1 - z0, w.ny, w.nx), dtype=torch.float64, pin_memory=True)
        if w.init == "tgv":
            a, b = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, z0, z1, w.nz, xp=torch,
                                    device=torch.device("cuda", local))
            rh.copy_(a)
            uh.copy_(b)
            del a, b
        else:
            a, b = synth.initial_fields(w, z0, z1, w.nz)
            rh.copy_(torch.from_numpy(a))
            uh.copy_(torch.from_numpy(b))
        ro = torch.empty_like(rh, pin_memory=True)
        uo = torch.empty_like(uh, pin_memory=True)
        rn, un, ron, uon = rh.numpy(), uh.numpy(), ro.numpy(), uo.numpy()
        barrier()
        t0 = time.perf_counter()
        lat.init_fields(rn, un)
        lat.step(args.steps)
        lat.get_macroscopic(out=(ron, uon))
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        nbytes = 4 * nloc * 8
        e2e = {"value": w.nodes * args.steps / e2e_s / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
               "note": "init_fields(host rho,u) + K steps + get_macroscopic(host), pinned buffers, "
                       "wall clock with device sync, max over ranks"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peaks()
    achieved = bpn * nodes_per_launch / (kernel_ms * 1e-3) / 1e9
    prec = "fp64" if w.precision == 0 else "fp32"
    kfull = lat.kernel_name()
    traffic, traffic_src = ncu_traffic(w.name, prec, kfull, nodes_per_launch)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "source_hash": kernel_source_hash(),
            "peak_source": peak_src,
            "kernel": kfull,
            "bytes_per_node": bpn, "nodes_per_launch": nodes_per_launch, "kernel_ms_mean": kernel_ms,
            "launches_timed": tk["launches"],
            "note": "achieved = 2*27*sizeof(real) B/node x nodes per launch / mean launch duration (library "
                    "CUDA events around each collide-stream launch on the compute stream, K steps after the "
                    "timed region; at N>1 a step has 2 launches: boundary planes + interior; with the fused P2P halo "
                    "one event pair spans both concurrent launches of a step)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, n, ws = oracle_mlups(w, budget_s=12.0)
        cpu = {"value": v, "unit": "MLUPS", "cores": 1, "kind": "oracle",
               "sample": f"{n} steps of {ws.nx}x{ws.ny}x{ws.nz} (same physics as {w.name}), single thread pinned to 1 core",
               "cpu_model": host_cpu()[0], "host_logical_cores": host_cpu()[1]}
    line = {"metric": METRIC, "value": mlups, "unit": "MLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.workload == "weak" else "strong", "vs_baseline": None,
            "dtype": "f64" if prec == "fp64" else "f64-arith/f32-storage", "data": "synthetic",
            "config": {"workload": w.name, "grid_global": [w.nx, w.ny, w.nz], "nodes_global": w.nodes,
                       "r": w.r, "s": w.s, "nu": w.nu, "corrections": args.corrections.upper(),
                       "collision": "3DCCM" if w.model == 0 else "3DCRM", "storage": prec,
                       "l2": ("working set per step >> 126 MB L2; no flush needed" if flush is None else
                              f"buffers ({lat.info()['buffer_bytes'] / 1e6:.1f} MB each) fit in L2: 512 MB L2 "
                              "flush (untimed) before every step, per-step CUDA events summed"),
                       "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                       "nccl_comm": dict(zip(("nranks", "rank"), lat.comm_ranks())),
                       "halo": {0: "in-kernel wrap", 1: "nccl ghost planes", 2: "fused p2p ghost planes"}[lat.info()["halo"]],
                       "streaming": aa_fit_note or ("AA in place (1 buffer)" if args.streaming == "aa" else "AB (2 buffers)")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "bad_nodes": bad}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dry_run(args):
    """The launch plan of this rank without a GPU (what a torchrun N-GPU run would
    do), and, with WORLD_SIZE > 1, the max-over-ranks aggregation of per-rank
    times over a gloo process group: rank 0 prints one JSON line."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    w = workload(args, world)
    z0, z1 = synth.slab_range(w.nz, rank, world)
    halo = ("in-kernel wrap" if world == 1 and args.halo == "auto" else
            "fused p2p ghost planes" if args.halo == "p2p" else "nccl ghost planes")
    launches_per_step = 1 if halo == "in-kernel wrap" else 2  # boundary planes + interior
    plan = {"rank": rank, "world": world, "workload": w.name, "grid_global": [w.nx, w.ny, w.nz],
            "slab": [z0, z1], "nodes_local": w.nx * w.ny * (z1 - z0), "halo": halo,
            "gpu_launches_timed": launches_per_step * args.steps}
    # a fake per-rank device time (ms) that differs between ranks; value = global nodes x K / max
    t = 10.0 + rank
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        x = torch.tensor([t], dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        t = float(x.item())
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        dist.destroy_process_group()
    else:
        plans = [plan]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": "weak" if args.workload == "weak" else "strong",
                          "max_rank_ms": t, "value": w.nodes * args.steps / (t * 1e-3) / 1e6, "plans": plans}),
              flush=True)


def main():
    args = parse()
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_cuda(args)


if __name__ == "__main__":
    main()
