"""CPU checks of the multi-GPU launch logic of bench.py and scripts/scale_sweep.sh
(no GPU): under torchrun with world sizes 2 and 4 each rank's z-slab, the
workload (weak: 512^3 per GPU; strong: 1024 x 1024 x 512 in total), the halo
mode and the launch count are what a GPU run would use, and the whole-job value
is global nodes x K / (max over ranks of the per-rank time), reduced over a gloo
process group."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(n, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(n), "--dry-run", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 4])
def test_weak_scaling_plan_and_aggregation(n):
    d = _torchrun(n, "--steps", "7")
    assert d["n_gpus"] == n and d["scaling"] == "weak"
    assert d["max_rank_ms"] == 10.0 + (n - 1)  # the slowest rank's (fake) time
    nodes = 512 * 512 * 512 * n
    assert d["value"] == pytest.approx(nodes * 7 / (d["max_rank_ms"] * 1e-3) / 1e6)
    slabs = [p["slab"] for p in sorted(d["plans"], key=lambda p: p["rank"])]
    assert slabs == [[512 * r, 512 * (r + 1)] for r in range(n)]
    assert all(p["grid_global"] == [512, 512, 512 * n] and p["halo"] == "nccl ghost planes" for p in d["plans"])
    assert all(p["gpu_launches_timed"] == 2 * 7 for p in d["plans"])


def test_strong_scaling_plan_p2p():
    d = _torchrun(4, "--workload", "strong", "--halo", "p2p", "--steps", "3")
    assert d["scaling"] == "strong"
    slabs = [p["slab"] for p in sorted(d["plans"], key=lambda p: p["rank"])]
    assert slabs == [[128 * r, 128 * (r + 1)] for r in range(4)]
    assert all(p["grid_global"] == [1024, 1024, 512] and p["halo"] == "fused p2p ghost planes" for p in d["plans"])


def test_scale_sweep_script_dry_run():
    env = dict(os.environ, DRY_RUN="1", PORT=str(_port()))
    r = subprocess.run(["bash", "scripts/scale_sweep.sh", "2"], capture_output=True, text=True, cwd=ROOT, env=env,
                       timeout=600)
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    # n = 1: weak auto, weak p2p, strong AA; n = 2: weak auto, weak p2p, strong auto, strong p2p
    assert [d["n_gpus"] for d in lines] == [1, 1, 1, 2, 2, 2, 2], r.stdout + r.stderr[-2000:]
    assert [d["scaling"] for d in lines] == ["weak", "weak", "strong", "weak", "weak", "strong", "strong"]
