"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/lbm_cuboid.h declares; host-side validation and the halo plan work
without a GPU (no compute calls here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lbm_cuboid.h")


@pytest.fixture(scope="module")
def P():
    from paper_2107_14774_b200 import build as B

    B.build()
    import paper_2107_14774_b200 as P

    P.load()
    return P


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lbm_cuboid_\w+)\s*\(", src)))


def test_header_symbols_exported(P):
    names = declared()
    assert len(names) >= 18
    assert sorted(P.lbm.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", P.lbm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lbm_cuboid_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    lib = P.load()
    for n in names:
        getattr(lib, n)


def test_library_is_sm100a_and_independent_of_oracle(P):
    out = subprocess.run(["cuobjdump", "--list-elf", P.lbm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", P.lbm.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "nccl" in ldd
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_2107_14774_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "cm_oracle" not in txt, f


def test_validation_errors(P):
    mk = P.lbm.make_params
    bb = P.lbm.buffer_bytes
    assert bb(mk(8, 4, 6, 1.0, 2.0, omega_nu=1.5)) == 27 * 8 * 4 * 8 * 8
    assert bb(mk(8, 4, 6, 1.0, 2.0, omega_nu=1.5, precision=1, world=2)) == 27 * 8 * 4 * 5 * 4
    bad = [dict(nx=0), dict(r=-1.0), dict(omega_nu=2.0), dict(omega_xi=0.0), dict(cs2=1.0),
           dict(bc=(1, 0, 0, 0, 0, 0)), dict(bc=(2, 2, 0, 0, 0, 0)), dict(world=4),
           dict(corrections=7), dict(omega_high=2.5)]
    for kw in bad:
        d = dict(nx=8, ny=4, nz=6, r=1.0, s=2.0, omega_nu=1.5)
        d.update(kw)
        with pytest.raises(P.LbmError) as ei:
            bb(mk(**d))
        assert ei.value.code == P.lbm.LBM_EINVAL
        assert P.load().lbm_cuboid_last_error().decode()


@pytest.mark.parametrize("world,bcz", [(1, 0), (2, 0), (4, 0), (3, 1)])
def test_halo_plan(P, world, bcz):
    nx, ny, nz = 5, 3, 12
    for rank in range(world):
        p = P.lbm.make_params(nx, ny, nz, 1.0, 2.0, omega_nu=1.5, world=world, rank=rank,
                              bc=(0, 0, 0, 0, bcz, bcz))
        hp = P.lbm.halo_plan(p)
        nxy, nzl = nx * ny, nz // world
        assert hp["ghost"] == (1 if world > 1 else 0)
        assert hp["count"] == 9 * nxy
        assert hp["send_up"] == nzl * 27 * nxy + 18 * nxy
        assert hp["recv_down"] == 18 * nxy
        assert hp["send_down"] == 27 * nxy
        assert hp["recv_up"] == (nzl + 1) * 27 * nxy
        if world > 1:
            up = (rank + 1) % world if (bcz == 0 or rank < world - 1) else -1
            dn = (rank - 1) % world if (bcz == 0 or rank > 0) else -1
            assert (hp["peer_up"], hp["peer_down"]) == (up, dn)
    p = P.lbm.make_params(nx, ny, nz, 1.0, 2.0, omega_nu=1.5, halo=1)
    hp = P.lbm.halo_plan(p)
    assert hp["ghost"] == 1 and hp["peer_up"] == 0 and hp["peer_down"] == 0


def test_c_example_compiles_against_the_header(P, tmp_path):
    """examples/tgv_c_abi.c uses only include/lbm_cuboid.h and the shared library."""
    exe = tmp_path / "tgv_c_abi"
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "tgv_c_abi.c"), "-o", str(exe),
                           "-L", os.path.dirname(P.lbm.LIB_PATH), "-l:liblbm_cuboid.so",
                           f"-Wl,-rpath,{os.path.dirname(P.lbm.LIB_PATH)}", "-lm"])
    assert exe.exists()


def test_params_struct_layout_matches_header(P, tmp_path):
    """The ctypes mirror of lbm_cuboid_params has the C struct's size and field
    offsets (gcc, from include/lbm_cuboid.h); LBM_P2P_BLOB_BYTES agrees."""
    fields = [f[0] for f in P.lbm.Params._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stddef.h>\n#include <stdio.h>\n#include \"lbm_cuboid.h\"\nint main(void) {\n"
                   "  printf(\"size %zu\\n\", sizeof(lbm_cuboid_params));\n"
                   "  printf(\"blob %d\\n\", LBM_P2P_BLOB_BYTES);\n"
                   + "".join(f"  printf(\"{f} %zu\\n\", offsetof(lbm_cuboid_params, {f}));\n" for f in fields)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).splitlines())
    import ctypes

    assert int(out.pop("size")) == ctypes.sizeof(P.lbm.Params)
    assert int(out.pop("blob")) == P.lbm.P2P_BLOB_BYTES
    for f in fields:
        assert int(out[f]) == getattr(P.lbm.Params, f).offset, f
    # every field of the C struct is mirrored (count the declarators in the header)
    hdr = re.sub(r"/\*.*?\*/", "", open(HDR).read(), flags=re.S)
    body = hdr[hdr.index("typedef struct {"):hdr.index("} lbm_cuboid_params;")]
    names = re.findall(r"[\s*](\w+)\s*(?:\[\d+\])?\s*[,;]", body)
    assert sorted(names) == sorted(fields), (sorted(names), sorted(fields))


def test_plane_size_limit(P):
    """27 nx ny must stay below 2^31 (int32 offsets within a plane): the largest
    accepted plane and the first rejected one."""
    lim = (2 ** 31 - 1) // 27
    nx = 8191
    ok_ny = lim // nx
    assert P.lbm.buffer_bytes(P.lbm.make_params(nx, ok_ny, 2, 1.0, 2.0, omega_nu=1.5)) > 0
    with pytest.raises(P.LbmError) as ei:
        P.lbm.buffer_bytes(P.lbm.make_params(nx, ok_ny + 1, 2, 1.0, 2.0, omega_nu=1.5))
    assert ei.value.code == P.lbm.LBM_EINVAL


def test_mode_validation(P):
    """Launch/halo/streaming mode fields: out-of-range values are LBM_EINVAL,
    unsupported combinations LBM_ENOTSUP (host-side, no GPU)."""
    mk, bb = P.lbm.make_params, P.lbm.buffer_bytes
    base = dict(nx=8, ny=4, nz=6, r=1.0, s=2.0, omega_nu=1.5)
    for kw, code in [(dict(halo=3), P.lbm.LBM_EINVAL), (dict(graphs=4), P.lbm.LBM_EINVAL),
                     (dict(graphs=-1), P.lbm.LBM_EINVAL), (dict(streaming=2), P.lbm.LBM_EINVAL),
                     (dict(model=2), P.lbm.LBM_EINVAL), (dict(precision=2), P.lbm.LBM_EINVAL),
                     (dict(streaming=1, halo=2), P.lbm.LBM_ENOTSUP),
                     (dict(streaming=1, halo=1), P.lbm.LBM_ENOTSUP),
                     (dict(streaming=1, world=2, rank=0), P.lbm.LBM_ENOTSUP),
                     (dict(streaming=1, corrections=3), P.lbm.LBM_ENOTSUP)]:
        d = dict(base)
        d.update(kw)
        with pytest.raises(P.LbmError) as ei:
            bb(mk(**d))
        assert ei.value.code == code, (kw, ei.value)
    # accepted: P2P with FULL_FD, the persistent launch mode, fp32 storage
    for kw in (dict(halo=2, corrections=3), dict(graphs=3), dict(precision=1, graphs=3)):
        d = dict(base)
        d.update(kw)
        assert bb(mk(**d)) > 0
