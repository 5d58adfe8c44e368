"""The ME_DEBUG build (libme_debug.so): the same kernels with a bounds check on every staged-
region load and visited-bitmap access (a failed check prints and traps).  The geometry and
trace parity suites run against it in a subprocess; compute-sanitizer is not available on the
GPU pool, so these checks stand in for memcheck on the shared-memory side."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_parity_suites_under_debug_checks():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    sys.path.insert(0, ROOT)
    from paper_0806_0689_b200 import build
    so = build.build(debug=True)
    env = dict(os.environ, ME_LIBRARY=so)
    chk = subprocess.run([sys.executable, "-c", "import paper_0806_0689_b200.me as m; m.load(); print(m.SO_PATH)"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert chk.stdout.strip().endswith("libme_debug.so"), chk.stdout + chk.stderr
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_geometry_gpu.py"),
                        os.path.join(ROOT, "tests", "test_trace_gpu.py"),
                        os.path.join(ROOT, "tests", "test_compact_gpu.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "passed" in r.stdout
