"""Bounds-checked run of every kernel (compute-sanitizer is closed on this pool):
a -DLBM_DEBUG_BOUNDS build of liblbm_cuboid.so checks every population load and
store of the collide-stream kernels against its buffer and reports violations
through lbm_cuboid_sync; scripts/sanitize_run.py exercises all kernels, models,
precisions, wall kinds, the NCCL ghost path and graphs on small grids."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_kernels():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2107_14774_b200 import build as B

    lib = os.path.join(ROOT, "build", "variants", "lib_debug.so")
    if not os.path.exists(lib) or any(os.path.getmtime(s) > os.path.getmtime(lib) for s in B.sources()):
        subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "sweep.py"), "build", "debug"])
    env = dict(os.environ, LBM_CUBOID_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all kernels exercised" in r.stdout


def test_bounds_checked_randomised_cases():
    """The 240 randomised parity cases (tests/test_gpu_fuzz.py) rerun on the
    bounds-checked build: every population access of every collide-stream
    kernel in range (lbm_cuboid_sync reports a violation as an error), and the
    results still match the oracle."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2107_14774_b200 import build as B

    lib = os.path.join(ROOT, "build", "variants", "lib_debug.so")
    if not os.path.exists(lib) or any(os.path.getmtime(s) > os.path.getmtime(lib) for s in B.sources()):
        subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "sweep.py"), "build", "debug"])
    env = dict(os.environ, LBM_CUBOID_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_fuzz.py"), "-q",
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
