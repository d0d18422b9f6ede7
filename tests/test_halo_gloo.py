"""World-size-2 (and 3) CPU test of the z-slab halo exchange over torch.distributed
(gloo): each rank holds its slab in the library's buffer layout (DESIGN.md
"Data layout": [z_local+1][q][y][x], q = (ex+1)+3(ey+1)+9(ez+1), ghost planes
at 0 and nz_l+1), exchanges exactly what lbm_cuboid_halo_plan() prescribes in
the prescribed order, and then the pull-streaming source of every direction of
every local node must equal the global (periodic or walled) pull source."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, bcz, result):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2107_14774_b200 as P

    nx, ny, nz = 4, 3, 6 * world
    p = P.lbm.make_params(nx, ny, nz, 1.0, 2.0, omega_nu=1.5, world=world, rank=rank,
                          bc=(0, 0, 0, 0, bcz, bcz))
    hp = P.lbm.halo_plan(p)
    nzl, nxy = nz // world, nx * ny
    rng = np.random.default_rng(0)
    glob = rng.normal(size=(nz, 27, ny, nx))            # post-collision state, internal q order
    buf = np.full((nzl + 2, 27, ny, nx), np.nan)
    buf[1:nzl + 1] = glob[rank * nzl:(rank + 1) * nzl]
    flat = torch.from_numpy(buf.reshape(-1))
    c = hp["count"]
    reqs, recvs = [], []
    if hp["peer_up"] >= 0:
        reqs.append(dist.isend(flat[hp["send_up"]:hp["send_up"] + c].clone(), hp["peer_up"]))
    if hp["peer_down"] >= 0:
        t = torch.empty(c, dtype=torch.float64)
        reqs.append(dist.irecv(t, hp["peer_down"]))
        recvs.append((hp["recv_down"], t))
    if hp["peer_down"] >= 0:
        reqs.append(dist.isend(flat[hp["send_down"]:hp["send_down"] + c].clone(), hp["peer_down"]))
    if hp["peer_up"] >= 0:
        t = torch.empty(c, dtype=torch.float64)
        reqs.append(dist.irecv(t, hp["peer_up"]))
        recvs.append((hp["recv_up"], t))
    for r in reqs:
        r.wait()
    for off, t in recvs:
        flat[off:off + c] = t
    buf = flat.numpy().reshape(nzl + 2, 27, ny, nx)
    ok = True
    for zl in range(nzl):
        zg = rank * nzl + zl
        for q in range(27):
            ez = q // 9 - 1
            zs = zg - ez
            if not (0 <= zs < nz) and bcz != 0:
                continue  # a wall: bounce-back inside the kernel, no ghost needed
            want = glob[zs % nz, q]
            got = buf[zl + 1 - ez, q]
            ok &= bool(np.array_equal(want, got))
    result[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("world,bcz", [(2, 0), (2, 1), (3, 0)])
def test_gloo_halo_exchange_matches_global_pull(world, bcz):
    from paper_2107_14774_b200 import build as B

    B.build()
    mgr = mp.Manager()
    res = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), bcz, res), nprocs=world, join=True,
                       start_method="spawn")
    assert dict(res) == {r: True for r in range(world)}


def _p2p_worker(rank, world, port, bcz, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2107_14774_b200 as P

    p = P.lbm.make_params(4, 3, 2 * world, 1.0, 2.0, omega_nu=1.5, world=world, rank=rank,
                          bc=(0, 0, 0, 0, bcz, bcz), halo=P.HALO_P2P)
    hp = P.lbm.halo_plan(p)
    blobs = [None] * world
    dist.all_gather_object(blobs, f"blob-of-rank-{rank}".encode())
    dn, up = P.lbm.p2p_neighbour_blobs(hp, blobs)
    plans = [None] * world
    dist.all_gather_object(plans, hp)
    ok = bool(hp["ghost"])
    # the blob picked for each side is the neighbour's own
    ok &= (dn is None) == (hp["peer_down"] < 0) and (up is None) == (hp["peer_up"] < 0)
    if dn is not None:
        ok &= dn == f"blob-of-rank-{hp['peer_down']}".encode()
    if up is not None:
        ok &= up == f"blob-of-rank-{hp['peer_up']}".encode()
    # symmetry: my up neighbour's down neighbour is me (its flag word [0] is mine)
    if hp["peer_up"] >= 0:
        ok &= plans[hp["peer_up"]]["peer_down"] == rank
    if hp["peer_down"] >= 0:
        ok &= plans[hp["peer_down"]]["peer_up"] == rank
    # the region a rank stores into its up neighbour (send_up) lands at the
    # neighbour's recv_down offset, plane nz_l above: same q block, ghost p = 0
    nxy, nzl = 12, 2
    ok &= hp["send_up"] - nzl * 27 * nxy == hp["recv_down"]
    ok &= hp["send_down"] + nzl * 27 * nxy == hp["recv_up"]
    result[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("world,bcz", [(2, 0), (3, 1), (4, 0)])
def test_gloo_p2p_neighbour_wiring(world, bcz):
    """Host logic of the fused P2P halo under a real process group: descriptor
    all-gather, neighbour selection from the halo plan, symmetric flag slots and
    the store offsets the boundary kernel uses."""
    from paper_2107_14774_b200 import build as B

    B.build()
    mgr = mp.Manager()
    res = mgr.dict()
    mp.start_processes(_p2p_worker, args=(world, _free_port(), bcz, res), nprocs=world, join=True,
                       start_method="spawn")
    assert dict(res) == {r: True for r in range(world)}
