"""The plain-C program examples/tgv_c_abi.c (no Python, no torch) drives the
library through the C ABI; its result equals the Python binding's (the C side
computes its initial fields with libm, so they may differ in the last ulp).""" 
import os
import subprocess

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_matches_python_binding(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    libdir = os.path.dirname(P.lbm.LIB_PATH)
    exe = tmp_path / "tgv_c_abi"
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "tgv_c_abi.c"), "-o", str(exe), "-L", libdir,
                           "-l:liblbm_cuboid.so", f"-Wl,-rpath,{libdir}", "-lm"])
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), "200", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    w = synth.CONFIGS["tgv"]
    g = P.Lattice(**w.params())
    rho, u = synth.initial_fields(w)
    g.init_fields(rho, u)
    g.step(200)
    rp, up = g.get_macroscopic()
    data = np.fromfile(out, dtype=np.float64)
    n = w.nodes
    assert np.abs(data[:n].reshape(rp.shape) - rp).max() < 1e-13
    assert np.abs(data[n:].reshape(up.shape) - up).max() < 1e-13
    assert '"mass_change"' in r.stdout


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_multi_gpu_example_runs_on_one_gpu(halo):
    """examples/multi_gpu_tgv.py under torchrun with one process: runs, and the
    kinetic energy decays at the linear Taylor-Green rate (within 10 %)."""
    import re
    import socket
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "examples", "multi_gpu_tgv.py"), "--halo", halo, "--grid", "128",
                        "--steps", "200"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    m = re.search(r"KE ratio ([0-9.]+) \(linear theory ([0-9.]+)\)", r.stdout)
    assert m, r.stdout
    import math

    # decay exponent within 10 % of linear theory (128 nodes, 200 steps: the
    # start-up acoustic transient of the TGV initial state is part of the KE)
    assert abs(math.log(float(m.group(1))) / math.log(float(m.group(2))) - 1.0) < 0.1
