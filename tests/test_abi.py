"""The C ABI library loads and exports every symbol include/me.h declares; arguments are
validated before any device work (no compute calls here: this runs without a GPU)."""
import ctypes
import os
import re

import pytest
import torch

import paper_0806_0689_b200 as pkg
from paper_0806_0689_b200 import build as me_build
from paper_0806_0689_b200 import me

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "me.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(me_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    me_build.build()
    return me.load()


def test_header_symbols_exported(lib):
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"libme.so does not export {n}"
    assert sorted(me.SYMBOLS) == names, "binding symbol list out of sync with include/me.h"


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump -lelf {me.SO_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_oracle_not_linked():
    """The product library shares no code with the oracle (no oracle symbol in libme.so)."""
    out = os.popen(f"nm -D {me.SO_PATH}").read()
    assert "oracle" not in out


def test_strerror(lib):
    assert lib.me_strerror(0) == b"ok"
    assert lib.me_strerror(-3).startswith(b"me_init")


@pytest.mark.parametrize("W,H,block,p,expect", [
    (176, 144, 16, 7, None),       # valid: only fails for lack of init
    (170, 144, 16, 7, -1),         # W % block
    (176, 144, 12, 7, -1),         # block not in {8,16}
    (176, 144, 16, 0, -1),         # p < 1
    (176, 144, 16, 33, -1),        # p > 32
    (168, 144, 8, 7, -2),          # W % 16
    (0, 144, 16, 7, -1),
])
def test_validation_before_device_work(lib, W, H, block, p, expect):
    buf = ctypes.create_string_buffer((1 << 20) + 64)
    base = (ctypes.addressof(buf) + 15) & ~15
    rc = lib.me_dcds(base, base, W, H, block, p, base, base, base)
    if expect is None:
        if torch.cuda.is_available():
            pytest.skip("a GPU process may already be initialised")
        assert rc == me.ME_ENOTINIT
    else:
        assert rc == expect


def test_misaligned_pointer(lib):
    buf = ctypes.create_string_buffer(1 << 16)
    base = ((ctypes.addressof(buf) + 15) & ~15) + 1
    assert lib.me_dcds(base, base - 1, 176, 144, 16, 7, base - 1, base - 1, base - 1) == me.ME_EALIGN


def test_null_pointers(lib):
    assert lib.me_dcds(None, None, 176, 144, 16, 7, None, None, None) == me.ME_EINVAL
    buf = ctypes.create_string_buffer(1 << 16)
    base = (ctypes.addressof(buf) + 15) & ~15
    assert lib.me_dcds_batch(base, base, 0, 0, 176, 144, 16, 7, base, base, base, None) == me.ME_EINVAL


def test_init_without_gpu_fails_loudly(lib):
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc = lib.me_init(0)
    assert rc in (me.ME_ECUDA, me.ME_EINVAL)
    with pytest.raises(pkg.MEError):
        pkg.me_init(0)


def test_no_cpu_fallback_in_binding():
    """The binding never imports the oracle or computes SADs itself."""
    src = open(os.path.join(ROOT, "paper_0806_0689_b200", "me.py")).read()
    assert "oracle" not in src
    for f in os.listdir(os.path.join(ROOT, "paper_0806_0689_b200")):
        if f.endswith(".py"):
            assert "import oracle" not in open(os.path.join(ROOT, "paper_0806_0689_b200", f)).read()
