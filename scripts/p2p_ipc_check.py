"""Multi-process check of the fused P2P halo's CUDA-IPC wiring on ONE GPU.

Launched with torchrun (gloo process group, every rank on cuda:0).  The ranks
export their P2P descriptors, all-gather them and map their neighbours'
population buffers and flag words through cudaIpcOpenMemHandle, exactly as on a
multi-GPU box.  The slabs are then stepped ONE RANK AT A TIME (host barrier
between ranks), so every flag a stream waits on is already set when the wait is
enqueued: no GPU work of one process ever waits on another process's work in
flight (B200_PROFILING.md: ranks sharing one GPU must not wait on one another).
Rank 0 compares the gathered slabs with an undecomposed lattice: bitwise.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29511 scripts/p2p_ipc_check.py [--case periodic|walls]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", choices=["periodic", "walls"], default="periodic")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    torch.cuda.set_device(0)
    if args.case == "periodic":
        w = synth.CONFIGS["tgv"].scaled(nx=20, ny=11, nz=4 * world)
    else:
        w = synth.CONFIGS["cavity100"].scaled(nx=13, ny=9, nz=3 * world)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 77)
    lat = P.distributed_lattice(device=0, halo=P.HALO_P2P, **w.params())
    assert lat.info()["halo"] == 2
    z0, z1 = synth.slab_range(w.nz, rank, world)

    def serial(fn):
        for r in range(world):
            if rank == r:
                fn()
                lat.sync()
            dist.barrier()

    serial(lambda: lat.init_fields(np.ascontiguousarray(rho[z0:z1]), np.ascontiguousarray(u[:, z0:z1])))
    for _ in range(args.steps):
        serial(lambda: lat.step(1))
    parts = [None] * world
    dist.all_gather_object(parts, lat.get_populations())
    ok = True
    if rank == 0:
        ref = P.Lattice(device=0, **w.params())
        ref.init_fields(rho, u)
        ref.step(args.steps)
        f_ref = ref.get_populations()
        ref.close()
        f = np.concatenate(parts, axis=1)
        ok = bool(np.array_equal(f, f_ref))
        print(json.dumps({"case": args.case, "world": world, "steps": args.steps, "bitwise_equal": ok,
                          "max_abs_diff": float(np.abs(f - f_ref).max())}))
    dist.barrier()
    lat.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
