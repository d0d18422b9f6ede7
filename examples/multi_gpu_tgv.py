"""Multi-GPU Taylor-Green vortex through the Python binding (one process per GPU).

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      examples/multi_gpu_tgv.py [--halo nccl|p2p] [--grid 256] [--steps 500]

Each rank owns a z-slab of an n x n x n/2 lattice (r = 1, s = 2: a cubic
physical box), initialises its slab of the decaying Taylor-Green vortex,
advances it, and the ranks reduce the kinetic energy, which is compared with
the linear decay exp(-6 nu k^2 t) (reading R9).
"""
import argparse
import math
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--halo", choices=["nccl", "p2p"], default="nccl")
    ap.add_argument("--grid", type=int, default=256, help="nodes along x and y (nz = grid/2)")
    ap.add_argument("--steps", type=int, default=500)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()

    w = synth.CONFIGS["weak"].scaled(nx=args.grid, ny=args.grid, nz=args.grid // 2, u0=1e-3)
    halo = P.HALO_P2P if args.halo == "p2p" else P.HALO_AUTO
    lat = P.distributed_lattice(device=local, halo=halo, **w.params())
    z0, z1 = synth.slab_range(w.nz, rank, world)
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, z0, z1, w.nz, xp=torch,
                              device=torch.device("cuda", local))
    lat.init_fields(rho, u)

    def kinetic_energy():
        out = torch.tensor([lat.check()["kinetic_energy"]], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(out)
        return float(out.item())

    e0 = kinetic_energy()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    start.record(lat.stream)
    lat.step(args.steps)
    end.record(lat.stream)
    lat.sync()
    ms = torch.tensor([start.elapsed_time(end)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    e1 = kinetic_energy()
    k = 2 * math.pi / w.nx
    theory = math.exp(-6 * w.nu * k * k * args.steps)
    if rank == 0:
        print(f"{world} GPU(s), {args.halo} halo, {w.nx}x{w.ny}x{w.nz}: {args.steps} steps in "
              f"{ms.item():.1f} ms = {w.nodes * args.steps / (ms.item() * 1e3):.0f} MLUPS; "
              f"KE ratio {e1 / e0:.6f} (linear theory {theory:.6f})")
    dist.barrier()
    lat.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
