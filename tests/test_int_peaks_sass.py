"""tools/int_peaks.cu (the ALU roofline denominator, profiles/int_peaks.json) measures what its
labels say: compiled for sm_100a, each variant's loop is the named SASS instruction (nothing
folded or merged away; VERDICT r1 found the old IADD3 leg folded).  CPU only (nvcc + cuobjdump)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = "/usr/local/cuda/bin/nvcc"

WANT = {0: "VABSDIFF4.U8.ACC", 1: "IDP.4A", 2: "SHF.R.W", 3: "PRMT", 4: "LOP3.LUT", 5: "IMAD",
        6: "IMAD.HI", 7: "IADD3"}


@pytest.fixture(scope="module")
def sass(tmp_path_factory):
    if not os.path.exists(NVCC):
        pytest.skip("no nvcc")
    cub = str(tmp_path_factory.mktemp("ip") / "ip.cubin")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin", "-o", cub,
                           os.path.join(ROOT, "tools", "int_peaks.cu")])
    out = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    funcs = {}
    for blk in out.split("Function : ")[1:]:
        m = re.match(r"_Z4kernILi(\d+)EEvPjijPx", blk.split()[0])
        if m:
            funcs[int(m.group(1))] = blk
    return funcs


@pytest.mark.parametrize("op", sorted(WANT))
def test_single_op_loops(sass, op):
    ins = [ln.split(";")[0].split("*/")[-1].strip() for ln in sass[op].splitlines() if "*/" in ln]
    n = sum(1 for i in ins if i.split()[0:1] and i.split()[0].startswith(WANT[op])
            and not (WANT[op] == "IMAD" and (i.startswith("IMAD.MOV") or i.startswith("IMAD.HI") or i.startswith("IMAD.WIDE"))))
    assert n >= 8 * 16, (op, n)  # the unrolled loop body: >= 16 iterations x 8 chains


@pytest.mark.parametrize("mix,other", [(15, "IMAD"), (17, "IADD3"), (12, "SHF.R.W"), (13, "PRMT")])
def test_mix_loops(sass, mix, other):
    body = sass[mix]
    assert body.count("VABSDIFF4.U8.ACC") >= 16 and body.count(other) >= 16
