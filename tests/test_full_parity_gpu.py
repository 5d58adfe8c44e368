"""Every pair of config c3 at full size (239 pairs of 1920x1088, 7.8 M blocks) bit-exact against
the oracle -- DCDS, DCDS^S and full search: mv / SAD / points of every block and the per-pair
statistics (tools/full_parity.py, the oracle in one process per host core).  The same tool over
c0-c4 and every algorithm (DCDS, DCDS^S, CDS, DS, h-/v-HEXBS, FS; all 959 2160p pairs of c4
except FS) is recorded in profiles/r2/full_parity.json: 34 sweeps, all bit-exact."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c3_every_pair_bit_exact(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    out = tmp_path / "fp.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "full_parity.py"), "--configs", "c3", "--algs", "dcds,dcds_s,fs",
                        "--out", str(out)], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ALL BIT-EXACT" in r.stdout
